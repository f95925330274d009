"""The MBU-Net forward on the GPU: model upload, planning, CUDA-graph replay.

``forward(model, image, threads=1, trace=False)`` is the drop-in for
``bitunet.graph.forward`` (``pkg/src/bitunet/graph.py:413-458``): same
arguments, same :class:`ForwardResult` (float64 logits, uint8 mask, and with
``trace=True`` a ``{name: {"acc", "out"}}`` dict whose bit outputs are
:class:`BitTensor` objects byte-identical to the reference's).

Underneath, :class:`DeviceModel` uploads each compiled layer once
(``mbu_conv_create`` repacks the w+/w- planes for the tensor cores) and hands
them to the native runner (``mbu_model_*``), which plans every activation as
a view into one workspace and enqueues the whole network on a stream.
:class:`Engine` adds persistent device buffers and a captured CUDA graph for
steady-state throughput (bench.py).
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref

import numpy as np
import torch

from . import _lib
from .bitcore import BitTensor, ChannelSegment, segment_lane_table, segment_lanes
from .errors import EngineError, ShapeError, UnsupportedConfigError
from .ops import ConvHandle, FloatConvHandle, _ptr, _stream, cuda_device

__all__ = ["DeviceModel", "Engine", "forward", "ForwardResult"]


def _result_cls():
    from .graph import ForwardResult

    return ForwardResult


ForwardResult = None  # resolved lazily (graph imports runtime lazily too)


class DeviceModel:
    """A compiled model resident on one GPU, driven by the native runner."""

    def __init__(self, model, device=None):
        self.device = cuda_device(device)
        self.config = model.config
        self.names, self.kinds = [], []
        self.out_segments = []  # per layer: output lane layout (bit layers)
        self.out_channels = []  # per layer: logical channel count
        self.concat_skip = {}  # concat layer -> its skip operand (the other one is the layer before)
        h = ctypes.c_void_p()
        _lib.call("mbu_model_create", ctypes.byref(h), self.device.index)
        self.handle = h
        index = {}
        segs = ()
        cur_c = model.config.in_channels
        seen_float = False
        with torch.cuda.device(self.device):
            for i, layer in enumerate(model.layers):
                kind = layer.kind
                if kind == "float-conv":
                    lanes = None
                    if seen_float or i > 0:
                        lanes = segment_lane_table(segs)
                    fc = FloatConvHandle(layer.weights, layer.bias, layer.spec,
                                         bn=layer.bn if layer.apply_sign else None,
                                         in_lanes=lanes, device=self.device)
                    _lib.call("mbu_model_add_fconv", h, fc.release(), int(bool(layer.apply_sign)))
                    seen_float = True
                    segs = (ChannelSegment(0, layer.spec.c_out),)
                    cur_c = layer.spec.c_out
                elif kind in ("binary-conv", "masked-conv", "binary-tconv", "masked-tconv"):
                    cv = ConvHandle(layer.weights, layer.spec, segs, layer.threshold,
                                    transposed=kind.endswith("tconv"), device=self.device)
                    _lib.call("mbu_model_add_conv", h, cv.release())
                    segs = (ChannelSegment(0, layer.spec.c_out),)
                    cur_c = layer.spec.c_out
                elif kind == "maxpool":
                    _lib.call("mbu_model_add_maxpool", h)
                elif kind == "concat":
                    j = index[layer.concat_with]
                    _lib.call("mbu_model_add_concat", h, j)
                    self.concat_skip[i] = j
                    shift = segment_lanes(segs)
                    segs = segs + tuple(ChannelSegment(s.lane_offset + shift, s.count)
                                        for s in self.out_segments[j])
                    cur_c = cur_c + self.out_channels[j]
                else:
                    raise UnsupportedConfigError(f"unknown layer kind {kind!r}")
                index[layer.name] = i
                self.names.append(layer.name)
                self.kinds.append(kind)
                self.out_segments.append(segs)
                self.out_channels.append(cur_c)
        self._finalizer = weakref.finalize(self, _destroy_model, h)
        self.planned = None
        self.ws_bytes = 0

    def plan(self, n, height, width, trace=False):
        key = (n, height, width, bool(trace))
        if self.planned == key:
            return self.ws_bytes
        size = ctypes.c_size_t()
        _lib.call("mbu_model_plan", self.handle, n, height, width, int(bool(trace)),
                  ctypes.byref(size))
        self.planned = key
        self.ws_bytes = int(size.value)
        return self.ws_bytes

    def run(self, image, logits, mask, workspace, path=_lib.PATH_AUTO, stream=None):
        """Enqueue one forward on ``stream`` (all arguments CUDA tensors)."""
        s = _stream(self.device) if stream is None else ctypes.c_void_p(stream.cuda_stream)
        # the native plan is per model handle: run only what it was planned for
        if self.planned is None or tuple(image.shape[:3]) != self.planned[:3]:
            raise EngineError(f"image {tuple(image.shape)} does not match the plan {self.planned}")
        _lib.call("mbu_forward", self.handle, _ptr(image), _ptr(logits), _ptr(mask),
                  _ptr(workspace), workspace.numel() * workspace.element_size(), path, s)

    def set_timing(self, enable: bool):
        """Record CUDA events around every layer of the next eager runs."""
        _lib.call("mbu_model_set_timing", self.handle, int(bool(enable)))

    def layer_times(self):
        """Per-layer durations (ms) of the last timed forward, on its stream."""
        out = (ctypes.c_float * len(self.names))()
        _lib.call("mbu_model_layer_times", self.handle, out)
        return list(out)

    def layer_info(self, i):
        vals = [ctypes.c_int() for _ in range(7)]
        ob, ab = ctypes.c_size_t(), ctypes.c_size_t()
        accc = ctypes.c_int()
        _lib.call("mbu_model_layer_info", self.handle, i, *[ctypes.byref(v) for v in vals],
                  ctypes.byref(ob), ctypes.byref(ab), ctypes.byref(accc))
        kind, n, h, w, cw, stride, off = (v.value for v in vals)
        nofs = ctypes.c_size_t(-1).value
        return dict(kind=kind, n=n, h=h, w=w, wpp=cw, stride=stride, offset=off,
                    out_off=None if ob.value == nofs else ob.value,
                    acc_off=None if ab.value == nofs else ab.value, acc_c=accc.value)

    def read_trace(self, workspace: torch.Tensor, logits_np: np.ndarray, frames=None) -> dict:
        """Assemble the reference trace dict from the planned workspace.

        ``frames`` (a slice of the batch axis) restricts the copy to those
        frames, sliced on the device: a full-size batch-8 trace is ~35 GB."""
        ws = workspace.view(torch.uint8)
        sel = slice(None) if frames is None else frames
        trace = {}
        for i, name in enumerate(self.names):
            info = self.layer_info(i)
            n, h, w = info["n"], info["h"], info["w"]
            n_sel = len(range(n)[sel])
            acc = None
            if info["acc_off"] is not None:
                c = info["acc_c"]
                is_f = self.kinds[i] == "float-conv"
                nbytes = n * h * w * c * (8 if is_f else 4)
                raw = ws[info["acc_off"]:info["acc_off"] + nbytes]
                acc = raw.view(torch.float64 if is_f else torch.int32).reshape(n, h, w, c)
                acc = acc[sel].cpu().numpy()
            if info["kind"] == 1:  # the head: float logits
                out = logits_np
                acc = logits_np
            elif i in self.concat_skip:
                # planned as a split view (no concat buffer): the reference's
                # concat words are operand a's words, then operand b's
                # (layers.py:369-384; wpp_a is whole 128-lane blocks)
                a, b = trace[self.names[i - 1]]["out"], trace[self.names[self.concat_skip[i]]]["out"]
                out = BitTensor(n_sel, h, w, self.out_channels[i],
                                np.ascontiguousarray(np.concatenate([a.words, b.words], axis=-1)),
                                self.out_segments[i])
            else:
                stride, off, wpp = info["stride"], info["offset"], info["wpp"]
                nbytes = n * h * w * stride * 8
                raw = ws[info["out_off"]:info["out_off"] + nbytes].view(torch.int64)
                words = raw.reshape(n, h, w, stride)[sel, ..., off:off + wpp].cpu().numpy()
                out = BitTensor(n_sel, h, w, self.out_channels[i],
                                np.ascontiguousarray(words).view(np.uint64),
                                self.out_segments[i])
            trace[name] = {"acc": acc, "out": out}
        return trace


def _destroy_model(h):
    if _lib._lib is not None:
        _lib.load().mbu_model_destroy(h)


_CACHE: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_STRONG: dict = {}


def _device_model(model, device) -> DeviceModel:
    dev = cuda_device(device)
    try:
        per_model = _CACHE.setdefault(model, {})
    except TypeError:  # not weak-referenceable: keep the model alive with its upload
        per_model = _STRONG.setdefault(id(model), (model, {}))[1]
    dm = per_model.get(dev)
    if dm is None:
        dm = per_model[dev] = DeviceModel(model, dev)
    return dm


_STAGE: dict = {}  # device index -> pinned float64 staging buffer of the drop-in forward's upload
_STAGE_LOCK = threading.Lock()


def _upload(image: np.ndarray, dev) -> torch.Tensor:
    """Host float64 array -> device tensor through a cached page-locked staging
    buffer, in chunks: the (multi-threaded) host copy of chunk k+1 overlaps the
    DMA of chunk k. A pageable ``.to()`` pushes both through the driver's small
    bounce buffers, several times slower for a 403 MB batch."""
    src = torch.from_numpy(np.ascontiguousarray(image)).reshape(-1)
    out = torch.empty(src.numel(), dtype=torch.float64, device=dev)
    chunk = 1 << 22  # 32 MB
    with _STAGE_LOCK:  # one staging buffer per device, shared by concurrent callers
        stage = _STAGE.get(dev.index)
        if stage is None or stage.numel() < src.numel():
            stage = torch.empty(src.numel(), dtype=torch.float64, pin_memory=True)
            _STAGE[dev.index] = stage
        for a in range(0, src.numel(), chunk):
            b = min(a + chunk, src.numel())
            stage[a:b].copy_(src[a:b])
            out[a:b].copy_(stage[a:b], non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()  # the staging buffer is free again
    return out.view(image.shape)


_STAGE_OUT: dict = {}  # device index -> pinned byte staging buffer of the results


def _download(ts, dev) -> list:
    """Device tensors -> ordinary numpy arrays: full-rate DMA into a cached
    page-locked buffer, then a multi-threaded host copy out of it (the results
    the caller keeps are not page-locked memory)."""
    nbytes = [t.numel() * t.element_size() for t in ts]
    with _STAGE_LOCK:
        stage = _STAGE_OUT.get(dev.index)
        if stage is None or stage.numel() < sum(nbytes):
            stage = torch.empty(sum(nbytes), dtype=torch.uint8, pin_memory=True)
            _STAGE_OUT[dev.index] = stage
        views, off = [], 0
        for t, nb in zip(ts, nbytes):
            v = stage[off:off + nb].view(t.dtype).view(t.shape)
            v.copy_(t, non_blocking=True)
            views.append(v)
            off += nb
        torch.cuda.current_stream(dev).synchronize()
        out = []
        for v in views:
            a = np.empty(tuple(v.shape), dtype=torch.empty(0, dtype=v.dtype).numpy().dtype)
            torch.from_numpy(a).copy_(v)
            out.append(a)
    return out


def _ws_budget() -> int:
    """Workspace bytes one forward() call may plan (MBU_FORWARD_WS_BYTES, default 32 GiB)."""
    return int(os.environ.get("MBU_FORWARD_WS_BYTES", 32 << 30))


def forward(model, image, threads: int = 1, trace: bool = False, *, device=None,
            path=_lib.PATH_AUTO):
    """Run the compiled network on an (n, H, W, C) float64 image, on the GPU.

    ``image`` is a host array (uploaded here) or a float64 CUDA tensor already
    on the device (e.g. from ``decode_raster``), used in place."""
    cfg = model.config
    on_dev = isinstance(image, torch.Tensor) and image.is_cuda
    if on_dev:
        if image.dtype != torch.float64:
            raise ShapeError(f"device image must be float64, got {image.dtype}")
        device = image.device if device is None else device
    else:
        image = np.asarray(image, dtype=np.float64)
    if image.ndim != 4 or tuple(image.shape[1:]) != (cfg.height, cfg.width, cfg.in_channels):
        raise ShapeError(
            f"image shape {tuple(image.shape)} != (n, {cfg.height}, {cfg.width}, {cfg.in_channels})")
    dm = _device_model(model, device)
    n = image.shape[0]
    dev = dm.device
    if not trace and n > 1:
        # frames are independent (the reference flattens them into M,
        # layers.py:276): a batch whose workspace would exceed the budget runs
        # as consecutive chunks of frames, which also keeps every conv input
        # under the engine's 2^31-word offsets
        step = max(1, _ws_budget() // max(1, dm.plan(1, cfg.height, cfg.width, False)))
        if n > step:
            parts = [forward(model, image[a:a + step], threads, False, device=dev, path=path)
                     for a in range(0, n, step)]
            return _result_cls()(np.concatenate([r.logits for r in parts]),
                                 np.concatenate([r.mask for r in parts]), None)
    ws_bytes = dm.plan(n, cfg.height, cfg.width, trace)
    with torch.cuda.device(dev):
        ws = torch.empty(max(ws_bytes, 8) // 8 + 1, dtype=torch.int64, device=dev)
        if on_dev:
            if image.device != dev:
                raise ShapeError(f"image is on {image.device}, model runs on {dev}")
            img = image.contiguous()
        else:
            img = _upload(image, dev)
        out_c = cfg.out_channels
        logits = torch.empty((n, cfg.height, cfg.width, out_c), dtype=torch.float64, device=dev)
        mask = torch.empty((n, cfg.height, cfg.width, out_c), dtype=torch.uint8, device=dev)
        dm.run(img, logits, mask, ws, path=path)
        logits_np, mask_np = _download([logits, mask], dev)
        notes = None
        if trace:
            notes = dm.read_trace(ws, logits_np)
            notes["mask"] = mask_np
    return _result_cls()(logits_np, mask_np, notes)


class Engine:
    """Steady-state executor: fixed batch, resident buffers, one CUDA graph.

    ``run()`` replays the captured forward on device-resident inputs;
    ``run_e2e(host_image, host_logits, host_mask)`` adds the pinned
    host->device image copy and the device->host logits/mask copies, the
    way a serving loop would use it.
    """

    def __init__(self, model, batch: int, device=None, use_graph: bool = True,
                 path=_lib.PATH_AUTO, with_logits: bool = True):
        cfg = model.config
        # an Engine owns its model handle: the native plan (batch, buffer
        # offsets) is per handle, so a forward() or another Engine on the same
        # model can never re-plan the buffers this Engine's graphs replay
        self.dm = DeviceModel(model, cuda_device(device))
        self.device = self.dm.device
        self.batch = batch
        self.shape = (batch, cfg.height, cfg.width, cfg.in_channels)
        self.out_shape = (batch, cfg.height, cfg.width, cfg.out_channels)
        ws_bytes = self.dm.plan(batch, cfg.height, cfg.width, False)
        dev = self.device
        with torch.cuda.device(dev):
            self.ws = torch.empty(max(ws_bytes, 8) // 8 + 1, dtype=torch.int64, device=dev)
            self.image = torch.zeros(self.shape, dtype=torch.float64, device=dev)
            self.logits = torch.empty(self.out_shape, dtype=torch.float64, device=dev)
            self.mask = torch.empty(self.out_shape, dtype=torch.uint8, device=dev)
            self.stream = torch.cuda.Stream(dev)
            self.path = path
            self.graph = None
            self.launches_per_run = None
            before = _lib.launch_count()
            with torch.cuda.stream(self.stream):
                self._enqueue()
            self.stream.synchronize()
            self.launches_per_run = _lib.launch_count() - before
            if use_graph:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self.stream):
                    self._enqueue()
                self.graph = g

    def _enqueue(self, image=None, logits=None, mask=None):
        self.dm.run(self.image if image is None else image,
                    self.logits if logits is None else logits,
                    self.mask if mask is None else mask, self.ws, path=self.path,
                    stream=torch.cuda.current_stream(self.device))

    # ------------------------------------------------------------ streaming
    def _ensure_slots(self):
        """Second set of I/O buffers + graph for copy/compute overlap."""
        if getattr(self, "_slots", None) is not None:
            return
        dev = self.device
        with torch.cuda.device(dev):
            slots = [(self.image, self.logits, self.mask, self.graph)]
            img = torch.zeros(self.shape, dtype=torch.float64, device=dev)
            lg = torch.empty(self.out_shape, dtype=torch.float64, device=dev)
            mk = torch.empty(self.out_shape, dtype=torch.uint8, device=dev)
            g = None
            if self.graph is not None:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self.stream):
                    self._enqueue(img, lg, mk)
            slots.append((img, lg, mk, g))
            self._slots = slots
            self.h2d = torch.cuda.Stream(dev)
            self.d2h = torch.cuda.Stream(dev)
            ev = lambda: torch.cuda.Event()  # noqa: E731
            self._ev = {k: [ev(), ev()] for k in ("h2d", "comp", "d2h")}
            self._used = [False, False]

    def run_stream(self, host_images, host_logits, host_masks, steps: int):
        """Pipelined serving loop over ``steps`` batches.

        Step i copies ``host_images[i % len]`` (pinned) to the device on a
        copy stream, runs the forward on the compute stream, and copies the
        logits / mask back on a second copy stream into
        ``host_logits[i % len]`` / ``host_masks[i % len]``. Two device buffer
        sets let step i+1's upload and step i-1's download overlap step i's
        compute. Returns after enqueueing; synchronize on ``self.d2h``.
        """
        self._ensure_slots()
        ev = self._ev
        for i in range(steps):
            s = i & 1
            img, lg, mk, g = self._slots[s]
            hi = host_images[i % len(host_images)]
            hl = None if host_logits is None else host_logits[i % len(host_logits)]
            hm = host_masks[i % len(host_masks)]
            with torch.cuda.stream(self.h2d):
                if self._used[s]:
                    self.h2d.wait_event(ev["comp"][s])  # slot's image consumed
                img.copy_(hi, non_blocking=True)
                ev["h2d"][s].record(self.h2d)
            with torch.cuda.stream(self.stream):
                self.stream.wait_event(ev["h2d"][s])
                if self._used[s]:
                    self.stream.wait_event(ev["d2h"][s])  # slot's outputs downloaded
                if g is not None:
                    g.replay()
                else:
                    self._enqueue(img, lg, mk)
                ev["comp"][s].record(self.stream)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(ev["comp"][s])
                if hl is not None:
                    hl.copy_(lg, non_blocking=True)
                hm.copy_(mk, non_blocking=True)
                ev["d2h"][s].record(self.d2h)
            self._used[s] = True

    def run_stream_raster(self, host_rasters, maxval: int, host_logits, host_masks, steps: int):
        """``run_stream`` for frame streams in netpbm sample form (SURVEY.md
        §8(f) rank 2): step i uploads the pinned uint8 raster
        ``host_rasters[i % len]`` of shape (batch, H, W, C) (or (batch, H, W, C, 2) for
        16-bit samples; 1-2 bytes per sample instead of 8), decodes it on the GPU into the image buffer
        (``decode_raster``: sample / maxval, the reference's read_image
        arithmetic), then runs the forward and downloads as ``run_stream``."""
        from .ops import decode_raster

        self._ensure_slots()
        rshape = tuple(host_rasters[0].shape)
        if rshape not in (self.shape, self.shape + (2,)):
            raise ShapeError(f"raster batches must be {self.shape} (+ (2,) for 16-bit), got {rshape}")
        if getattr(self, "_raster_slots", None) is None or tuple(self._raster_slots[0].shape) != rshape:
            self._raster_slots = [torch.empty(rshape, dtype=torch.uint8, device=self.device)
                                  for _ in range(2)]
        ev = self._ev
        for i in range(steps):
            s = i & 1
            img, lg, mk, g = self._slots[s]
            rs = self._raster_slots[s]
            hr = host_rasters[i % len(host_rasters)]
            hl = None if host_logits is None else host_logits[i % len(host_logits)]
            hm = host_masks[i % len(host_masks)]
            with torch.cuda.stream(self.h2d):
                if self._used[s]:
                    self.h2d.wait_event(ev["comp"][s])
                rs.copy_(hr, non_blocking=True)
                ev["h2d"][s].record(self.h2d)
            with torch.cuda.stream(self.stream):
                self.stream.wait_event(ev["h2d"][s])
                if self._used[s]:
                    self.stream.wait_event(ev["d2h"][s])
                decode_raster(rs, maxval, out=img)
                if g is not None:
                    g.replay()
                else:
                    self._enqueue(img, lg, mk)
                ev["comp"][s].record(self.stream)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(ev["comp"][s])
                if hl is not None:
                    hl.copy_(lg, non_blocking=True)
                hm.copy_(mk, non_blocking=True)
                ev["d2h"][s].record(self.d2h)
            self._used[s] = True

    def run(self):
        with torch.cuda.stream(self.stream):
            if self.graph is not None:
                self.graph.replay()
            else:
                self._enqueue()

    def run_e2e(self, host_image: torch.Tensor, host_logits: torch.Tensor | None,
                host_mask: torch.Tensor):
        with torch.cuda.stream(self.stream):
            self.image.copy_(host_image, non_blocking=True)
            if self.graph is not None:
                self.graph.replay()
            else:
                self._enqueue()
            if host_logits is not None:
                host_logits.copy_(self.logits, non_blocking=True)
            host_mask.copy_(self.mask, non_blocking=True)
