"""Per-group role timeline of CTA 0 for one layer launch (debug; see tac_debug_set_trace).
Needs a trace build: TACSNN_TRACE=1 python -m paper_2603_13810_b200.build --force.

    python scripts/trace_layer.py --layer 0 --B 256
Prints, per group iteration, the producer / MMA / epilogue event times (us, relative).
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2603_13810_b200 import configs, tacsnn  # noqa: E402

NAMES = ["prod_start", "prod_done", "mma_ready", "mma_issued", "epi_full", "epi_released", "epi_done",
         "prod_raw", "prod_issued", "mma_afull", "mma_refill", "p1_start", "p1_done", "p1_raw"]
SHOW = [0, 1, 7, 11, 12, 13, 9, 10, 2, 3, 4, 5, 6]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--layer", type=int, default=0)
    ap.add_argument("--B", type=int, default=256)
    ap.add_argument("--rows", type=int, default=24)
    ap.add_argument("--mode", default=None)
    ap.add_argument("--K", type=int, default=None)
    ap.add_argument("--npw", type=int, default=3, help="warp-stage producer warps (5 on OCC=2 first layers)")
    a = ap.parse_args()
    cfg = configs.CONFIGS[a.config]
    spec = configs.layer_plan(cfg, mode=a.mode, K=a.K, B=a.B)[a.layer]
    w, b = configs.layer_weights(cfg)[a.layer]
    prep = tacsnn.prepare_weights(spec, w, b)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = tacsnn.pack((torch.rand((spec.T, spec.B, spec.C_in, spec.H, spec.W), device="cuda",
                                generator=g) < 0.15).to(torch.uint8))
    tacsnn.conv_lif(spec, prep, x)  # warm
    buf = torch.zeros(4096 * 16, dtype=torch.int64, device="cuda")
    tacsnn.lib().tac_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
    tacsnn.conv_lif(spec, prep, x)
    torch.cuda.synchronize()
    tacsnn.lib().tac_debug_set_trace(None)
    tr = buf.view(4096, 16).cpu().numpy()
    n = int((tr[:, 0] > 0).sum())
    t0 = tr[0, 0]
    print(f"layer {a.layer} B={a.B}: {n} group iterations traced on CTA 0")
    print("it " + " ".join(f"{NAMES[j]:>11s}" for j in SHOW))
    for i in list(range(min(a.rows, n))) + list(range(max(a.rows, n - 4), n)):
        print(f"{i:3d} " + " ".join(f"{(tr[i, j] - t0) / 1e3 if tr[i, j] else float('nan'):11.2f}" for j in SHOW))
    import numpy as np
    it = tr[1:n]
    d = lambda j0, j1: np.median(it[:, j1] - it[:, j0]) / 1e3
    per = np.median(np.diff(tr[:n, 6])) / 1e3
    print(f"median per-group period (epi_done diff): {per:.2f} us")
    print(f"median producer busy: {d(0, 1):.2f} us, MMA ready->issued: {d(2, 3):.2f} us, "
          f"epi full->released: {d(4, 5):.2f} us, epi released->done: {d(5, 6):.2f} us")
    print(f"MMA: prev issued -> A-full {np.median(tr[1:n, 9] - tr[:n-1, 3]) / 1e3:.2f} us, A-full -> refilled "
          f"{np.median(tr[:n, 10] - tr[:n, 9]) / 1e3:.2f} us, refilled -> ready (t_empty) {np.median(tr[:n, 2] - tr[:n, 10]) / 1e3:.2f} us; "
          f"CTA 1 producer done - CTA 0 producer done {np.median(tr[:n, 12] - tr[:n, 1]) / 1e3:.2f} us")
    print(f"median epi wait (prev done -> full): {np.median(tr[1:n, 4] - tr[:n-1, 6]) / 1e3:.2f} us; "
          f"MMA wait (prev issued -> ready): {np.median(tr[1:n, 2] - tr[:n-1, 3]) / 1e3:.2f} us; "
          f"producer wait (prev done -> start): {np.median(tr[1:n, 0] - tr[:n-1, 1]) / 1e3:.2f} us")
    # warp-stage producers (first layers): stage it is built by the warp that built it - npw
    w = a.npw
    if n > w + 1:
        print(f"  per producer warp (stage it vs it-{w}): raw wait {np.median(tr[w:n, 7] - tr[:n-w, 1]) / 1e3:.2f} us, "
              f"A-stage wait {np.median(tr[w:n, 0] - tr[w:n, 7]) / 1e3:.2f} us, "
              f"stage-to-stage {np.median(tr[w:n, 1] - tr[:n-w, 1]) / 1e3:.2f} us")
    print(f"  of which prev done -> raw ready: {np.median(tr[1:n, 7] - tr[:n-1, 1]) / 1e3:.2f} us, "
          f"raw ready -> A stage free: {np.median(tr[1:n, 0] - tr[1:n, 7]) / 1e3:.2f} us")


if __name__ == "__main__":
    main()
