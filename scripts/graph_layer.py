"""Kernel time of one layer without host overhead: N launches captured in a CUDA graph,
replayed and timed with CUDA events (for the small, launch-bound first layers).

    python scripts/graph_layer.py --config C3 --layer 0 --mode tac --K 8 --B 1024 [--n 20]
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
    ap.add_argument("--config", default="C3")
    ap.add_argument("--layer", type=int, default=0)
    ap.add_argument("--B", type=int, default=1024)
    ap.add_argument("--mode", default=None)
    ap.add_argument("--K", type=int, default=None)
    ap.add_argument("--n", type=int, default=20)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    cfg = configs.CONFIGS[a.config]
    spec = configs.layer_plan(cfg, mode=a.mode, K=a.K, B=a.B)[a.layer]
    w, b = configs.layer_weights(cfg)[a.layer]
    prep = tacsnn.prepare_weights(spec, w, b)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = tacsnn.pack((torch.rand((spec.T, spec.B, spec.C_in, spec.H, spec.W), device="cuda",
                                generator=g) < 0.15).to(torch.uint8))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        out, _, _ = tacsnn.conv_lif(spec, prep, x, want_counts=False)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            for _ in range(a.n):
                tacsnn.conv_lif(spec, prep, x, out=out, want_counts=False)
        graph.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            graph.replay()
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / a.n)
    print(f"layer {a.layer} {spec} engine={spec.engine_used()}")
    print("  graph us/launch: " + " ".join(f"{1e3 * t:.1f}" for t in ts))


if __name__ == "__main__":
    main()
