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
    def __init__(self, specs: list[LayerSpec], weights, device="cuda", voters: int | None = None):
        """voters: the VotingLayer size of the DVS network (10); None for the
        spike-count readout (MNIST/FMNIST)."""
        assert len(specs) == len(weights)
        self.specs = list(specs)
        self.voters = voters
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

    def readout(self, counts_last: torch.Tensor) -> torch.Tensor:
        """Class scores of the network from the last layer's spike counts [B, C_out]: the
        VotingLayer (tac_vote: each class's voters' mean firing rate) when the network has
        voters, else the firing rates count / T_out."""
        last = self.specs[-1]
        T_out = last.out_shape()[0]
        if self.voters:
            return tacsnn.vote(counts_last, self.voters, T_out)
        return tacsnn.vote(counts_last, 1, T_out)

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


class TrainableNetwork(Network):
    """The same stack for training: every layer runs
    tac_conv_lif_forward_train with its pool as a separate tac_or_pool2 (the backward
    needs the pre-pool spikes), and backward() chains tac_conv_lif_backward and
    tac_or_pool2_backward from the last layer to the first.  The plans are the
    inference plans (the image does not depend on out_pool)."""

    def __init__(self, specs, weights, device="cuda", surrogate="fast_sigmoid", alpha=25.0,
                 detach_reset=False):
        super().__init__(specs, weights, device)
        self.surrogate, self.alpha, self.detach = surrogate, alpha, detach_reset

    def forward_train(self, x: torch.Tensor):
        """Returns (final spikes, final counts, tape)."""
        B = x.shape[1]
        tape = []
        cnt = None
        n = len(self.specs)
        for i, (spec, prep) in enumerate(zip(self.specs, self.prepared)):
            s = (spec if spec.B == B else spec.replace(B=B)).replace(out_pool=1)
            x = flatten_for(s, x)
            out, _, cnt, y = tacsnn.conv_lif_train(s, prep, x, want_counts=(i == n - 1))
            tape.append((s, prep, x, y, out, spec.out_pool))
            hc, wc = s.conv_hw
            x = tacsnn.or_pool2(out, s.C_out, wc) if spec.out_pool == 2 else out
        return x, cnt, tape

    def backward(self, tape, g_out: torch.Tensor, prepool: bool = True):
        """g_out: dL/ds of the last layer's output spikes, fp32 [T_out,B,H,W,C] -- the
        unpooled spikes the count readout reads (prepool=True, H,W = H',W') or, if the last
        layer pools, the pooled map (prepool=False).  Returns the per-layer gradient dicts
        (first layer first)."""
        grads = [None] * len(tape)
        g = g_out
        for i in range(len(tape) - 1, -1, -1):
            s, prep, x, y, out, pool = tape[i]
            if pool == 2 and not (prepool and i == len(tape) - 1):
                # g is w.r.t. the pooled map: route it back through the OR-pool
                hc, wc = s.conv_hw
                g = tacsnn.or_pool2_backward(out, g.reshape(out.shape[0], s.B, hc // 2, wc // 2, s.C_out),
                                             s.C_out, wc)
            r = tacsnn.conv_lif_backward(s, prep, x, y, g.reshape(out.shape[0], s.B, *s.conv_hw, s.C_out),
                                         surrogate=self.surrogate, alpha=self.alpha,
                                         detach_reset=self.detach, want_input_grad=i > 0)
            grads[i] = r
            g = r["g_input"]
        return grads
