"""A stack of Conv-LIF layers run through libtacsnn, one ABI call per layer.

The spike tensors stay packed and resident in HBM between layers; each layer's
fused 2x2 OR-pool output is the next layer's input.  Batch shards are plain
views (the ABI takes the T and B strides), so the multi-GPU driver just hands
each rank its slice.
"""
from __future__ import annotations

import torch

from . import tacsnn
from .tacsnn import LayerSpec


def flatten_for(spec: LayerSpec, x: torch.Tensor) -> torch.Tensor:
    """A fully connected layer is a 1x1 conv of a 1x1 image: its packed input row is the
    previous layer's whole (H, W, C) map, i.e. the packed rows concatenated (a view when
    every row is a whole number of words)."""
    if spec.H == 1 and spec.W == 1 and x.shape[2] != 1:
        assert spec.C_in == x.shape[2] * x.shape[3] * 32, "rows must be whole words"
        x = x.reshape(x.shape[0], x.shape[1], 1, x.shape[2] * x.shape[3])
    return x


class Network:
    def __init__(self, specs: list[LayerSpec], weights, device="cuda"):
        assert len(specs) == len(weights)
        self.specs = list(specs)
        self.device = torch.device(device)
        self.prepared = [tacsnn.prepare_weights(s, w, b, device=self.device)
                         for s, (w, b) in zip(self.specs, weights)]

    def engines(self):
        return [s.engine_used() for s in self.specs]

    def forward(self, x: torch.Tensor, keep: bool = False, want_v_final: bool = False,
                want_counts: bool | str = "last"):
        """x: packed int32 [T, B, H, WPR] on the device.  Returns (final spikes,
        per-layer counts, per-layer outputs if keep, per-layer v_final if asked).
        want_counts: True (every layer), "last" (only the final layer's spike-count
        readout; the others are None) or False."""
        B = x.shape[1]
        counts, outs, vfs = [], [], []
        n = len(self.specs)
        for i, (spec, prep) in enumerate(zip(self.specs, self.prepared)):
            s = spec if spec.B == B else spec.replace(B=B)
            wc = want_counts is True or (want_counts == "last" and i == n - 1)
            x = flatten_for(s, x)
            x, vf, cnt = tacsnn.conv_lif(s, prep, x, want_v_final=want_v_final, want_counts=wc)
            counts.append(cnt)
            vfs.append(vf)
            if keep:
                outs.append(x)
        return x, counts, outs, vfs

    def capture(self, x: torch.Tensor):
        """Record one forward on the static input buffer `x` as a CUDA graph (the
        launch-bound small configs: one graph replay instead of 2 launches and a
        host round of argument checks per layer).  Returns (graph, outputs of
        forward); replaying the graph refreshes the outputs in place."""
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            self.forward(x)                      # warm-up outside the capture
        torch.cuda.current_stream(self.device).wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            outs = self.forward(x)
        return graph, outs

    def launches_per_forward(self) -> int:
        """Kernels one forward launches (measured from the library's counter)."""
        return self._launches

    def count_launches(self, x, want_counts: bool | str = "last"):
        """Kernels one forward (same counts policy as forward) launches."""
        n = 0
        B = x.shape[1]
        nl = len(self.specs)
        for i, (spec, prep) in enumerate(zip(self.specs, self.prepared)):
            s = spec if spec.B == B else spec.replace(B=B)
            wc = want_counts is True or (want_counts == "last" and i == nl - 1)
            x = flatten_for(s, x)
            x, _, _ = tacsnn.conv_lif(s, prep, x, want_counts=wc)
            n += tacsnn.last_launch_count()
        self._launches = n
        return n
