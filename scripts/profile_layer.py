"""Run one layer of a config a few times (for ncu / quick timing on the GPU box).

    python scripts/profile_layer.py --config C5 --layer 1 --B 256 --iters 3 [--engine tcgen05]
Prints the CUDA-event time per launch of the layer call.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2603_13810_b200 import configs, tacsnn  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--layer", type=int, default=1)
    ap.add_argument("--B", type=int, default=256)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--engine", default="auto")
    ap.add_argument("--mode", default=None)
    ap.add_argument("--K", type=int, default=None)
    ap.add_argument("--no-counts", action="store_true", help="as the bench (counts on the last layer only)")
    a = ap.parse_args()
    cfg = configs.CONFIGS[a.config]
    specs = configs.layer_plan(cfg, mode=a.mode, K=a.K, B=a.B, engine=a.engine)
    spec = specs[a.layer]
    w, b = configs.layer_weights(cfg)[a.layer]
    prep = tacsnn.prepare_weights(spec, w, b)
    g = torch.Generator(device="cuda").manual_seed(0)
    dense = (torch.rand((spec.T, spec.B, spec.C_in, spec.H, spec.W), device="cuda", generator=g)
             < 0.15).to(torch.uint8)
    x = tacsnn.pack(dense)
    del dense
    out = None
    times = []
    for _ in range(a.iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out, _, cnt = tacsnn.conv_lif(spec, prep, x, out=out, want_counts=not a.no_counts)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    hc, wc = spec.conv_hw
    G = spec.T // (1 if spec.mode == "dense" else spec.K)
    flops = 2.0 * spec.C_out * hc * wc * spec.C_in * 9 * G * spec.B
    print(f"layer {a.layer} {spec} engine={spec.engine_used()}")
    for t in times:
        rate = "" if cnt is None else f"rate {cnt.sum().item() / (spec.B * spec.C_out * hc * wc * spec.T):.4f}"
        print(f"  {t:.3f} ms  useful {flops / t / 1e9:.1f} TFLOP/s  {rate}")


if __name__ == "__main__":
    main()
