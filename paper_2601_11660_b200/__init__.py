"""B200-native MBU-Net inference engine, drop-in for ``bitunet``'s forward path.

The reference (arXiv 2601.11660's ``bitunet`` 0.1.0, a CPU NumPy/Numba
package) defines the model and layer API this package keeps: the
masked-binary conv layer, the MBU-Net forward call, and the w+/w- weight /
packed-activation layouts. Here the data-parallel path runs as hand-written
sm_100a CUDA kernels behind the C-ABI of ``include/mbunet.h``
(``libmbunet.so``), driven from PyTorch for device memory, streams and CUDA
graphs. There is no CPU fallback.

Host-side (build-time) pieces — config, topology, weight packing, BN
folding, bundle synthesis — are restatements of the reference's so models
can be built on machines without ``bitunet``; models built BY ``bitunet``
are accepted unchanged.
"""

__version__ = "0.1.0"

from .bitcore import (
    BitPlane,
    BitTensor,
    ChannelSegment,
    MaskedWeightPlanes,
    PackedBitMatrix,
    pack_bipolar,
    pack_bits_tensor,
    pack_tensor,
    unpack_bipolar,
    unpack_tensor,
)
from .errors import (
    BundleError,
    CudaError,
    EngineError,
    FormatError,
    LayoutError,
    PlaneOverlapError,
    ShapeError,
    UnsupportedConfigError,
    ValueAlphabetError,
)
from .graph import (
    ALL_LABELS,
    CONFIGURABLE_LABELS,
    CompiledLayer,
    CompiledModel,
    ForwardResult,
    PrecisionMap,
    UNetConfig,
    build,
    forward,
    input_segments,
    layer_specs,
    scale_config,
    validate,
)
from .layers import (
    CONST_NEG,
    CONST_POS,
    DIR_GE,
    DIR_LE,
    ConvSpec,
    FusedThreshold,
    concat_channels,
    fuse_bn_sign,
    pack_conv_weights,
    unpack_conv_weights,
    weight_position_sums,
)
from .imageio import read_image, read_raster, write_gray, write_mask
from .ops import (
    apply_threshold,
    argmax_classes,
    decode_raster,
    bit_gemm,
    conv_forward,
    float_bn_sign,
    float_conv,
    maxpool2,
    transposed_conv_forward,
    xor_popcount_rows,
)
from .quantizer import (
    BundleEntry,
    WeightBundle,
    dense_records,
    live_bundle,
    quantize_bundle,
    synthesize_bundle,
)
from .modelfile import read_model, read_tensor, write_model, write_tensor
from .runtime import DeviceModel, Engine

__all__ = [
    "__version__",
    "BitPlane", "BitTensor", "ChannelSegment", "MaskedWeightPlanes", "PackedBitMatrix",
    "pack_bipolar", "pack_bits_tensor", "pack_tensor", "unpack_bipolar", "unpack_tensor",
    "BundleError", "CudaError", "EngineError", "FormatError", "LayoutError",
    "PlaneOverlapError", "ShapeError", "UnsupportedConfigError", "ValueAlphabetError",
    "ALL_LABELS", "CONFIGURABLE_LABELS", "CompiledLayer", "CompiledModel", "ForwardResult",
    "PrecisionMap", "UNetConfig", "build", "forward", "input_segments", "layer_specs",
    "scale_config", "validate",
    "CONST_NEG", "CONST_POS", "DIR_GE", "DIR_LE", "ConvSpec", "FusedThreshold",
    "concat_channels", "fuse_bn_sign", "pack_conv_weights", "unpack_conv_weights",
    "weight_position_sums",
    "read_image", "read_raster", "write_gray", "write_mask", "decode_raster",
    "apply_threshold", "argmax_classes", "bit_gemm", "conv_forward", "float_bn_sign", "float_conv", "maxpool2",
    "transposed_conv_forward", "xor_popcount_rows",
    "BundleEntry", "WeightBundle", "dense_records", "live_bundle", "quantize_bundle",
    "synthesize_bundle",
    "read_model", "read_tensor", "write_model", "write_tensor",
    "DeviceModel", "Engine",
]
