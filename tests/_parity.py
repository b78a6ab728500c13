"""Parity helpers: run a layer through the C ABI and check it against the oracle
with the replay protocol.

  * spikes: bit-exact wherever |V - v_th| > band (1e-3 v_th, north_star; reading D9); inside the
    band the oracle takes the device's decision (excused) and continues, so
    after a zero-mismatch replay the oracle's own output equals the device's.
  * v_final: |V_dev - V_oracle| <= 1e-3 * max(|V_oracle|, v_th) elementwise.
  * counts: equal to the oracle's spike counts (exact).
  * pooled output: equal to the oracle's OR-pool of its own output (exact).
Stacks chain ORACLE outputs into the next oracle layer and DEVICE outputs into
the next device layer; the two are asserted equal at every boundary.
"""
import numpy as np
import torch

BAND = 1e-3
VTOL = 1e-3
# membranes must stay well inside the tolerance, not just under it: the largest
# |V_dev - V_oracle| / (1e-3 max(|V|, v_th)) of any layer is asserted <= HEADROOM
# (DESIGN.md section 4 error budget: int8 slices ~0.1, fp16 hi + lo paths ~1e-3)
HEADROOM = 0.5


def to_u32(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().contiguous().numpy().view(np.uint32)


def check_layer(T, O, spec, S_u8: np.ndarray, w, b, *, x_packed=None, v_init=None,
                label="", workspace=True):
    """Run `spec` on the device and the oracle; returns (oracle output u8
    [T_out,B,C,Hq,Wq] after the spec's pool, device output packed tensor as
    stored with the spec's pool, stats)."""
    assert S_u8.dtype == np.uint8
    s1 = spec.replace(out_pool=1)
    if x_packed is None:
        x_packed = T.pack(torch.from_numpy(S_u8).cuda())
    vi_dev = None
    if v_init is not None:   # oracle layout [B,C,H',W'] -> device [B,H',W',C]
        vi_dev = torch.from_numpy(np.ascontiguousarray(
            v_init.transpose(0, 2, 3, 1)).astype(np.float32)).cuda()
    prep = T.prepare_weights(spec, w, b)
    out, vf, cnt = T.conv_lif(s1, prep, x_packed, v_init=vi_dev, want_v_final=True, workspace=workspace)
    torch.cuda.synchronize()
    hc, wc = s1.conv_hw
    D = O.unpack_spikes(to_u32(out), s1.C_out, wc)
    r = O.forward(S_u8, w.numpy(), None if b is None else b.numpy(), K=s1.K, mode=s1.mode,
                  beta=s1.beta, v_th=s1.v_th, v_reset=s1.v_reset, reset=s1.reset,
                  stride=s1.stride, pad=s1.pad, partial=s1.partial,
                  v_init=None if v_init is None else v_init.astype(np.float32).astype(np.float64),
                  replay=D, band=BAND * s1.v_th, alpha=s1.agg_weights)
    assert r["mismatch"] == 0, f"{label}: {r['mismatch']} out-of-band spike mismatches " \
                               f"({r['excused']} excused of {D.size})"
    assert np.array_equal(r["out"], D)
    v_dev = vf.cpu().numpy().transpose(0, 3, 1, 2).astype(np.float64)
    v_ref = r["v_final"]
    err = np.abs(v_dev - v_ref)
    tol = VTOL * np.maximum(np.abs(v_ref), s1.v_th)
    assert np.all(err <= tol), f"{label}: v_final max err {err.max():.3e} " \
                               f"(worst ratio {(err / tol).max():.3f})"
    assert (err / tol).max() <= HEADROOM, f"{label}: v_final error uses {(err / tol).max():.3f} of the " \
                                          f"tolerance (headroom {HEADROOM})"
    assert np.array_equal(cnt.cpu().numpy().astype(np.int64), r["counts"]), f"{label}: counts"
    ref_out = r["out"]
    dev_out = out
    if spec.out_pool == 2:
        ref_out = O.or_pool2(r["out"])
        dev_out, _, _ = T.conv_lif(spec, prep, x_packed, v_init=vi_dev, want_counts=False)
        torch.cuda.synchronize()
        Dp = O.unpack_spikes(to_u32(dev_out), spec.C_out, wc // 2)
        assert np.array_equal(Dp, ref_out), f"{label}: pooled output != OR-pool(oracle)"
    stats = dict(rate=float(D.mean()), excused=r["excused"], n=int(D.size),
                 max_verr=float(err.max()), max_ratio=float((err / tol).max()), counts=r["counts"])
    return ref_out, dev_out, stats


def check_stack(T, O, specs, weights, S_u8, label=""):
    """Layer-by-layer parity of a stack; returns per-layer stats."""
    x_dev = None
    S = S_u8
    stats = []
    for i, (spec, (w, b)) in enumerate(zip(specs, weights)):
        if spec.H == 1 and spec.W == 1 and S.shape[-1] != 1:
            # fully connected layer: the (h, w, c)-ordered flattening of the previous map,
            # which is the device's packed row layout (x*C + c, rows concatenated)
            Tn, Bn = S.shape[:2]
            S = np.ascontiguousarray(S.transpose(0, 1, 3, 4, 2).reshape(Tn, Bn, -1, 1, 1))
            x_dev = x_dev.reshape(x_dev.shape[0], x_dev.shape[1], 1, -1)
        ref_out, dev_out, st = check_layer(T, O, spec, S, w, b, x_packed=x_dev,
                                           label=f"{label} layer {i}")
        stats.append(st)
        S, x_dev = ref_out, dev_out
    return stats
