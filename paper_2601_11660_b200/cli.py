"""Command-line front end for the GPU path: ``infer`` and ``bench`` with
``--device``, mirroring the reference's
``bitunet.cli`` flags and exit codes (pkg/src/bitunet/cli.py:3-13, :268-288,
:348-373, :474-499). The other reference subcommands (quantize, profile,
plan, analyze, verify) are host-side tooling outside the hot path.

    python -m paper_2601_11660_b200 infer --model m.mbun --image x.ppm \\
        --mask-out m.pgm --logits-out l.rten [--device cuda:0]
    python -m paper_2601_11660_b200 bench [--model m.mbun] [--extent HxW] \\
        [--batch B] [--reps R] [--device cuda:0]

``infer`` reads the netpbm samples on the host, decodes them on the GPU
(``decode_raster``, bit-identical to ``read_image``) and runs the forward on
the device image; outputs are byte-identical to the reference's.
``--threads`` is accepted for command-line compatibility and ignored (the
GPU path has no host worker pool).
"""

from __future__ import annotations

import argparse
import sys
import time

import numpy as np

from . import __version__
from .errors import (
    EngineError,
    FormatError,
    LayoutError,
    PlaneOverlapError,
    ShapeError,
    UnsupportedConfigError,
    ValueAlphabetError,
)

_INTERNAL_EXIT, _FORMAT_EXIT, _CONFIG_EXIT, _SHAPE_EXIT = 1, 3, 4, 5


def _extent(text: str):
    """``N`` or ``HxW`` (cli.py:228-239); the config checks divisibility."""
    parts = text.lower().split("x")
    try:
        vals = [int(p) for p in parts]
    except ValueError as exc:
        raise argparse.ArgumentTypeError(f"bad extent {text!r}") from exc
    if len(vals) == 1:
        vals = vals * 2
    if len(vals) != 2:
        raise argparse.ArgumentTypeError(f"extent must be N or HxW, got {text!r}")
    return tuple(vals)


def _cmd_infer(args) -> int:
    from .imageio import read_raster, write_mask
    from .modelfile import read_model, write_tensor
    from .ops import decode_raster
    from .runtime import forward

    model = read_model(args.model)
    raster, maxval = read_raster(args.image)
    cfg = model.config
    shape = raster.shape[1:4]
    if shape != (cfg.height, cfg.width, cfg.in_channels):
        raise ShapeError(f"image {args.image} has shape {shape}, model wants "
                         f"({cfg.height}, {cfg.width}, {cfg.in_channels})")
    image = decode_raster(raster, maxval, device=args.device)
    result = forward(model, image)
    if args.mask_out:
        if cfg.out_channels != 1:
            raise UnsupportedConfigError(
                f"mask output needs a 1-channel head, model has {cfg.out_channels}")
        write_mask(args.mask_out, result.mask[0, :, :, 0])
        print(f"wrote {args.mask_out}")
    if args.logits_out:
        write_tensor(args.logits_out, np.asarray(result.logits, dtype=np.float64))
        print(f"wrote {args.logits_out}")
    return 0


def _cmd_bench(args) -> int:
    import torch

    from .graph import UNetConfig, build
    from .quantizer import live_bundle
    from .modelfile import read_model
    from .runtime import Engine

    if args.model:
        model = read_model(args.model)
        if args.extent and args.extent != (model.config.height, model.config.width):
            raise ShapeError(f"model {args.model} is compiled for "
                             f"{model.config.height}x{model.config.width}, not {args.extent}")
    else:
        h, w = args.extent or (512, 512)
        cfg = UNetConfig(height=h, width=w)
        model = build(cfg, live_bundle(cfg, np.random.default_rng(0)))
    eng = Engine(model, batch=args.batch, device=args.device)
    eng.image.uniform_()
    for _ in range(2):
        eng.run()
    torch.cuda.synchronize(eng.device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(eng.stream)
    for _ in range(args.reps):
        eng.run()
    e1.record(eng.stream)
    torch.cuda.synchronize(eng.device)
    wall = time.perf_counter() - t0
    ms = e0.elapsed_time(e1) / args.reps
    cfg = model.config
    fps = args.batch / (ms / 1e3)
    if args.csv:
        print("extent,batch,ms_per_batch,frames_per_s,kernels_per_batch")
        print(f"{cfg.height}x{cfg.width},{args.batch},{ms:.4f},{fps:.2f},{eng.launches_per_run}")
    else:
        print(f"{cfg.height}x{cfg.width} batch {args.batch} on {eng.device}: {ms:.3f} ms/batch, "
              f"{fps:.1f} frames/s ({eng.launches_per_run} kernels per batch, "
              f"{args.reps} reps in {wall:.2f} s wall)")
    return 0


def _add_common(p):
    p.add_argument("--device", default=None, help="CUDA device (default: the current one)")
    p.add_argument("--threads", type=int, default=None,
                   help="accepted for compatibility with the CPU engine; ignored")


def _build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="paper_2601_11660_b200",
        description="MBU-Net forward on B200 (sm_100a): infer and bench.")
    parser.add_argument("--version", action="version", version=f"%(prog)s {__version__}")
    sub = parser.add_subparsers(dest="command", required=True, metavar="command")

    p = sub.add_parser("infer", help="run a model on an image")
    p.add_argument("--model", required=True, help="model file (.mbun)")
    p.add_argument("--image", required=True, help="input image (P5 PGM or P6 PPM)")
    p.add_argument("--mask-out", default=None, help="write the mask as P5 {0,255}")
    p.add_argument("--logits-out", default=None, help="write raw logits (f64 tensor file)")
    _add_common(p)
    p.set_defaults(handler=_cmd_infer)

    p = sub.add_parser("bench", help="device throughput of the forward")
    p.add_argument("--model", default=None, help="model file (default: built-in architecture, "
                                                 "random weights)")
    p.add_argument("--extent", type=_extent, default=None, help="N or HxW (default 512)")
    p.add_argument("--batch", type=int, default=8, help="frames per forward")
    p.add_argument("--reps", type=int, default=10, help="timed forwards")
    p.add_argument("--csv", action="store_true", help="comma-separated output")
    _add_common(p)
    p.set_defaults(handler=_cmd_bench)
    return parser


# Exit-code contract of the reference CLI (pkg/src/bitunet/cli.py:474-503), as a
# table: the first row whose classes match the raised exception wins.
_EXIT_TABLE = (
    ((FormatError, OSError), _FORMAT_EXIT, "error"),
    ((UnsupportedConfigError, ValueAlphabetError, PlaneOverlapError), _CONFIG_EXIT, "error"),
    ((ShapeError, LayoutError), _SHAPE_EXIT, "error"),
    ((EngineError,), _INTERNAL_EXIT, "error"),
    ((Exception,), _INTERNAL_EXIT, "internal error"),
)


def _exit_code(exc: BaseException) -> int:
    for classes, code, label in _EXIT_TABLE:
        if isinstance(exc, classes):
            detail = str(exc) if label == "error" else f"{type(exc).__name__}: {exc}"
            print(f"{label}: {detail}", file=sys.stderr)
            return code
    raise exc


def main(argv=None) -> int:
    """CLI entry; returns the process exit code (usage errors: argparse's 2)."""
    parser = _build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as stop:
        return int(stop.code or 0)
    try:
        return args.handler(args)
    except Exception as exc:  # noqa: BLE001 - mapped through _EXIT_TABLE
        return _exit_code(exc)


if __name__ == "__main__":
    sys.exit(main())
