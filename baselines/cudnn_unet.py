"""cuDNN FP16 U-Net with MBU-Net's exact topology — the paper's speed baseline.

The paper compares MBU-Net against an FP16 U-Net of the same shape
(SURVEY.md §8(d) "cuDNN FP16"). This module builds that
network from the channel schedule of ``graph.layer_specs``: every bit conv
becomes Conv2d(3x3) + ReLU with batchnorm folded into the conv bias (eval),
every transposed conv ConvTranspose2d(2x2, s2) + ReLU, pools MaxPool2d(2),
concat torch.cat, the head a 1x1 conv. Run in float16, channels_last,
cudnn.benchmark, captured in a CUDA graph — the strongest stock-PyTorch
configuration. Random weights: only the speed is compared.
"""

from __future__ import annotations

import torch
from torch import nn


class FP16UNet(nn.Module):
    def __init__(self, cfg):
        super().__init__()
        from paper_2601_11660_b200.graph import layer_specs

        self.steps = []
        mods = nn.ModuleDict()
        for e in layer_specs(cfg):
            key = e.name.replace(".", "_").replace("-", "_")
            if e.kind in ("float-conv", "bit-conv"):
                s = e.conv
                mods[key] = nn.Conv2d(s.c_in, s.c_out, s.kernel_h, s.stride, s.padding, bias=True)
            elif e.kind == "bit-tconv":
                s = e.conv
                mods[key] = nn.ConvTranspose2d(s.c_in, s.c_out, s.kernel_h, s.stride, bias=True)
            self.steps.append((e.name, e.kind, key, e.concat_with))
        self.mods = mods
        self.pool = nn.MaxPool2d(2)

    def forward(self, x):
        outs = {}
        for name, kind, key, skip in self.steps:
            if kind in ("float-conv", "bit-conv", "bit-tconv"):
                x = self.mods[key](x)
                if name != "head":
                    x = torch.relu(x)
            elif kind == "maxpool":
                x = self.pool(x)
            elif kind == "concat":
                x = torch.cat([x, outs[skip]], dim=1)
            outs[name] = x
        return x


class CudnnUNetRunner:
    """Batch-fixed FP16 U-Net forward replayed from a CUDA graph.

    ``fused=True`` is the stronger baseline: the same network through
    ``torch.compile`` (Inductor keeps cuDNN for the convolutions and fuses the
    bias / ReLU / concat traffic around them into generated kernels), then
    captured in the same CUDA graph. Only the baseline is compiled; the MBU-Net
    path never is.
    """

    def __init__(self, cfg, batch: int, device, fused: bool = False):
        torch.backends.cudnn.benchmark = True
        torch.backends.cudnn.allow_tf32 = True
        self.device = device
        self.net = FP16UNet(cfg).to(device).half().to(memory_format=torch.channels_last).eval()
        if fused:
            self.net = torch.compile(self.net, dynamic=False)
        self.x = torch.randn(batch, cfg.in_channels, cfg.height, cfg.width, device=device,
                             dtype=torch.float16).to(memory_format=torch.channels_last)
        self.stream = torch.cuda.Stream(device)
        with torch.no_grad(), torch.cuda.stream(self.stream):
            for _ in range(3):  # cudnn autotune + warm-up outside the graph
                self.y = self.net(self.x)
        self.stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.no_grad(), torch.cuda.graph(self.graph, stream=self.stream):
            self.y = self.net(self.x)

    def run(self):
        with torch.cuda.stream(self.stream):
            self.graph.replay()
