"""One small layer per operand path and engine, for compute-sanitizer.

    compute-sanitizer --tool memcheck  python scripts/sanitize.py
    compute-sanitizer --tool racecheck python scripts/sanitize.py --quick
    compute-sanitizer --tool synccheck python scripts/sanitize.py --quick

Every case runs through the C ABI (libtacsnn.so) on cuda:0 and synchronises, so
an error is attributed to the case printed just before it.  No oracle: the
sanitizer checks memory accesses, shared-memory hazards and barrier use only
(parity is tests/test_gpu_parity.py).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2603_13810_b200 import synth, tacsnn as T  # noqa: E402

# name, spec kwargs (tcgen05 operand path in the comment)
CASES = [
    ("int8_tma_c128", dict(T=4, B=2, C_in=128, H=16, W=16, C_out=128, pad=1, K=2, mode="tactp",
                           beta=0.5, out_pool=2)),                      # PATH_HALO, TMA raw halo
    ("int8_ldg_c32", dict(T=4, B=2, C_in=32, H=13, W=13, C_out=64, pad=0, K=2, mode="tac",
                          beta=0.5, out_pool=1)),                       # PATH_HALO, LDG producer
    ("int8_c96_c96", dict(T=4, B=2, C_in=96, H=10, W=9, C_out=96, pad=1, K=2, mode="tac",
                          beta=0.5, out_pool=2)),
    ("int8_cout8", dict(T=4, B=2, C_in=32, H=12, W=12, C_out=8, pad=1, K=4, mode="tactp",
                        beta=0.5, out_pool=1)),                         # atomic sub-word output
    ("h16_tma_c2", dict(T=4, B=2, C_in=2, H=32, W=32, C_out=128, pad=1, K=4, mode="tactp",
                        beta=0.5, out_pool=2)),                         # PATH_H16 packed, U in TMEM
    ("h16_ldg_c1", dict(T=8, B=2, C_in=1, H=28, W=28, C_out=32, pad=0, K=4, mode="tac",
                        beta=0.5, out_pool=2)),
    ("split_ldg_c1", dict(T=8, B=2, C_in=1, H=28, W=28, C_out=32, pad=0, K=4, mode="tac",
                          beta=0.9, out_pool=2)),                       # PATH_SPLIT, LUT
    ("split_tma_c32", dict(T=8, B=2, C_in=32, H=12, W=16, C_out=64, pad=1, K=4, mode="tac",
                           beta=0.9, out_pool=2)),
    ("generic_delayed", dict(T=4, B=2, C_in=32, H=12, W=12, C_out=32, pad=1, K=2, mode="tactp",
                             beta=0.5, reset="delayed", v_reset=-0.2, out_pool=2)),
    ("partial_T10K4", dict(T=10, B=2, C_in=32, H=12, W=16, C_out=64, pad=1, K=4, mode="tactp",
                           beta=0.5, out_pool=2, partial=True)),
]
REAL_CASES = [
    ("real_c2", dict(T=8, B=2, C_in=2, H=32, W=32, C_out=128, pad=1, K=4, mode="tac", beta=0.5,
                     out_pool=2, input="real")),
]


def run(name, kw, engine, real=False):
    spec = T.LayerSpec(**kw).replace(engine=engine)
    try:
        used = spec.engine_used()
    except RuntimeError:
        print(f"skip {name}/{engine} (outside envelope)", flush=True)
        return
    print(f"case {name}/{used}", flush=True)
    w, b = synth.weights(1, spec.C_out, spec.C_in, gain=2.0)
    prep = T.prepare_weights(spec, w, b)
    g = torch.Generator().manual_seed(3)
    if real:
        x = torch.rand((spec.T, spec.B, spec.H, spec.W, spec.C_in), generator=g).cuda()
    else:
        x = T.pack((torch.rand((spec.T, spec.B, spec.C_in, spec.H, spec.W), generator=g) < 0.2)
                   .to(torch.uint8).cuda())
    hc, wc = spec.conv_hw
    vi = torch.rand((spec.B, hc, wc, spec.C_out), generator=g).cuda() * 0.5
    out, vf, cnt = T.conv_lif(spec, prep, x, v_init=vi, want_v_final=True)
    torch.cuda.synchronize()
    print(f"  ok rate={cnt.sum().item() / max(1, out.numel())}", flush=True)


FC_CASES = [
    ("fc_1600_128", dict(T=8, B=130, C_in=1600, H=1, W=1, C_out=128, R=1, S=1, pad=0, K=4, mode="tac", beta=0.9)),
    ("fc_512_110", dict(T=8, B=3, C_in=512, H=1, W=1, C_out=110, R=1, S=1, pad=0, K=4, mode="tactp", beta=0.5)),
]
TRAIN_CASES = [   # training forward + backward: tcgen05 dgrad / wgrad, first-layer wgrad, FC GEMMs
    ("train_c128", dict(T=4, B=2, C_in=128, H=16, W=16, C_out=128, pad=1, K=2, mode="tactp", beta=0.5)),
    ("train_c2", dict(T=4, B=2, C_in=2, H=32, W=32, C_out=128, pad=1, K=2, mode="tac", beta=0.5)),
    ("train_fc", dict(T=4, B=3, C_in=512, H=1, W=1, C_out=110, R=1, S=1, pad=0, K=2, mode="tactp", beta=0.5)),
]


def run_fc(name, kw, workspace):
    spec = T.LayerSpec(**kw)
    print(f"case {name}/{spec.engine_used()}/ws={workspace}", flush=True)
    w, b = synth.weights(1, spec.C_out, spec.C_in, 1, 1, gain=3.0)
    prep = T.prepare_weights(spec, w, b)
    g = torch.Generator().manual_seed(3)
    x = T.pack((torch.rand((spec.T, spec.B, spec.C_in, 1, 1), generator=g) < 0.2).to(torch.uint8).cuda())
    out, vf, cnt = T.conv_lif(spec, prep, x, want_v_final=True, workspace=workspace)
    torch.cuda.synchronize()
    votes = T.vote(cnt, 10, spec.T) if spec.C_out % 10 == 0 else None
    torch.cuda.synchronize()
    print(f"  ok rate={cnt.sum().item() / max(1, out.numel())} vote={votes is not None}", flush=True)


def run_train(name, kw):
    spec = T.LayerSpec(**kw, out_pool=1)
    r = spec.R
    print(f"case {name}/{spec.engine_used()}", flush=True)
    w, b = synth.weights(1, spec.C_out, spec.C_in, r, r, gain=3.0)
    prep = T.prepare_weights(spec, w, b)
    g = torch.Generator().manual_seed(3)
    x = T.pack((torch.rand((spec.T, spec.B, spec.C_in, spec.H, spec.W), generator=g) < 0.2).to(torch.uint8).cuda())
    out, _, _, y = T.conv_lif_train(spec, prep, x)
    hc, wc = spec.conv_hw
    gs = torch.randn((out.shape[0], spec.B, hc, wc, spec.C_out), generator=g).cuda()
    res = T.conv_lif_backward(spec, prep, x, y, gs, surrogate="arctan", alpha=2.0, detach_reset=True)
    torch.cuda.synchronize()
    print(f"  ok |gW|={res['g_weight'].abs().sum().item():.3e}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="tcgen05 engine only, fewer cases")
    a = ap.parse_args()
    engines = ["tcgen05"] if a.quick else ["tcgen05", "simt"]
    cases = CASES[:6] if a.quick else CASES
    for eng in engines:
        for name, kw in cases:
            run(name, kw, eng)
        for name, kw in REAL_CASES:
            run(name, kw, eng, real=True)
    for name, kw in FC_CASES:
        for ws in (True, False):
            run_fc(name, kw, ws)
    for name, kw in TRAIN_CASES:
        run_train(name, kw)
    print("sanitize: all cases ran", flush=True)


if __name__ == "__main__":
    main()
