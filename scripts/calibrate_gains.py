"""Calibrate per-layer weight gains with the ORACLE (run once; results frozen in
paper_2603_13810_b200/configs.py GAINS).  Uses only oracle/ and the seeded input
generators -- no CUDA path.

For each layer in order, bisect (in log space) the gain g of
synth.weights(..., gain=g) so that the layer's output firing rate in the
config's primary mode is ~target; the layer's (pooled) oracle output is the next
layer's input.

    python scripts/calibrate_gains.py C4 --B 2 --target 0.1
"""
import argparse
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2603_13810_b200 import configs, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--B", type=int, default=2)
    ap.add_argument("--target", type=float, default=0.1)
    ap.add_argument("--iters", type=int, default=8)
    ap.add_argument("--mode", default=None, help="calibrate for this mode instead of the config's primary one")
    ap.add_argument("--head", action="store_true",
                    help="keep the frozen conv gains and calibrate the FC head (network_plan)")
    a = ap.parse_args()
    if a.head:
        return calibrate_head(a)
    cfg = configs.CONFIGS[a.config]
    if a.mode:
        cfg = dataclasses_replace(cfg, mode=a.mode)
    x = configs.make_inputs(cfg, B=a.B).numpy()
    t = cfg.T
    gains = []
    for i, L in enumerate(cfg.layers):
        K = 1 if cfg.mode == "dense" else min(cfg.K, t)
        lo, hi = 0.25, 16.0
        best = None
        for _ in range(a.iters):
            g = math.sqrt(lo * hi)
            w, b = synth.weights(cfg.seeds[0] * 1000 + i, L.C_out, L.C_in, 3, 3, gain=g)
            r = O.forward(x, w.numpy(), b.numpy(), K=K, mode=cfg.mode, beta=cfg.beta, pad=L.pad)
            rate = float(r["out"].mean())
            best = (g, rate, r["out"])
            print(f"  layer {i} gain {g:.3f} rate {rate:.4f}", flush=True)
            if rate < a.target:
                lo = g
            else:
                hi = g
        g, rate, out = best
        gains.append(round(g, 2))
        print(f"layer {i}: gain {g:.3f} -> rate {rate:.4f}", flush=True)
        x = O.or_pool2(out) if L.pool == 2 else out
        if cfg.mode == "tac":
            t //= K
    print("GAINS", gains)


def dataclasses_replace(cfg, **kw):
    import dataclasses
    return dataclasses.replace(cfg, **kw)


def calibrate_head(a):
    """FC head gains: the conv stack runs with its frozen gains, its (pooled) output is
    flattened in (h, w, c) order (the packed row layout) and each FC layer's gain is bisected."""
    cfg = configs.CONFIGS[a.config]
    if a.mode:
        cfg = dataclasses_replace(cfg, mode=a.mode)
    specs = configs.network_plan(cfg, B=a.B)
    weights = configs.layer_weights(cfg, mode=cfg.mode)
    x = configs.make_inputs(cfg, B=a.B).numpy()
    nconv = len(cfg.layers)
    for s, (w, b) in zip(specs[:nconv], weights):
        r = O.forward(x, w.numpy(), b.numpy(), K=s.K, mode=s.mode, beta=s.beta, pad=s.pad,
                      partial=s.partial)
        x = O.or_pool2(r["out"]) if s.out_pool == 2 else r["out"]
        print(f"  conv rate {float(r['out'].mean()):.4f}", flush=True)
    Tn, Bn = x.shape[:2]
    x = np.ascontiguousarray(x.transpose(0, 1, 3, 4, 2).reshape(Tn, Bn, -1, 1, 1))
    gains = []
    for i, s in enumerate(specs[nconv:]):
        lo, hi = 0.25, 32.0
        best = None
        for _ in range(a.iters):
            g = math.sqrt(lo * hi)
            w, b = synth.weights(cfg.seeds[0] * 1000 + 10 + i, s.C_out, s.C_in, 1, 1, gain=g)
            r = O.forward(x, w.numpy(), b.numpy(), K=s.K, mode=s.mode, beta=s.beta, pad=0,
                          partial=s.partial)
            rate = float(r["out"].mean())
            best = (g, rate, r["out"])
            print(f"  FC {i} gain {g:.3f} rate {rate:.4f}", flush=True)
            lo, hi = (g, hi) if rate < a.target else (lo, g)
        g, rate, out = best
        gains.append(round(g, 2))
        x = out
    print("FC GAINS", gains)


if __name__ == "__main__":
    main()
