"""Pins of the oracle's backward pass (oracle/tac_oracle.c tac_oracle_backward;
surrogate-gradient BPTT, PAPER.md:237 and App. E)
against things other than itself:

  * no-spike regime: with v_th out of reach the layer is LINEAR in W, b, v_init, the
    (continuous) input and the aggregation weights, so central finite differences of
    the oracle's own forward are exact up to rounding -- and the BPTT gradient of
    L = <c, V_final> must equal them;
  * an independent torch implementation: the forward written from Eq. (1) / Alg. 1 /
    Alg. 2 with F.conv2d and a spike function whose backward is the autograd
    derivative of the surrogate's smooth primitive (fast sigmoid: u / (1 + a|u|),
    snnTorch; arctan: arctan(pi/2 a u) / pi), differentiated by torch.autograd --
    all modes, both surrogates, detached and attached reset, learnable alpha.
"""
import zlib

import numpy as np
import pytest
import torch
import torch.nn.functional as F


def _fd_exact(rng, shape, scale=1.0):
    """values on a 2^-12 grid: x +- 2^-10 stays exact in fp32"""
    return (np.round(rng.uniform(-scale, scale, shape) * 4096) / 4096).astype(np.float32)


@pytest.mark.parametrize("mode,K", [("dense", 1), ("tac", 2), ("tactp", 3)])
def test_backward_no_spike_equals_finite_differences(oracle_mod, mode, K):
    O = oracle_mod
    rng = np.random.default_rng(3)
    T, B, Cin, H, W, Cout = 6, 2, 2, 5, 6, 3
    X = rng.random((T, B, Cin, H, W))                     # continuous input: dX is defined
    Wt, b = _fd_exact(rng, (Cout, Cin, 3, 3)), _fd_exact(rng, Cout, 0.2)
    alpha = _fd_exact(rng, K) if mode != "dense" else None
    vi = rng.standard_normal((B, Cout, H, W))
    c = rng.standard_normal((B, Cout, H, W))             # L = <c, V_final>
    kw = dict(K=K, mode=mode, beta=0.75, v_th=1e6, pad=1)

    def L(X_=X, W_=Wt, b_=b, vi_=vi, a_=alpha):
        r = O.forward(X_, W_, b_, v_init=vi_, alpha=a_, **kw)
        assert r["out"].sum() == 0
        return float((c * r["v_final"]).sum())

    T_out = T // K if mode == "tac" else T
    g = O.backward(X, Wt, b, np.zeros((T_out, B, Cout, H, W)), v_init=vi, g_vfinal=c, alpha=alpha,
                   detach_reset=True, **kw)
    e = 2.0 ** -10
    for idx in [(0, 0, 0, 0), (2, 1, 1, 2), (1, 0, 2, 1)]:
        Wp, Wm = Wt.copy(), Wt.copy()
        Wp[idx] += e
        Wm[idx] -= e
        assert g["g_W"][idx] == pytest.approx((L(W_=Wp) - L(W_=Wm)) / (2 * e), rel=1e-9, abs=1e-9)
    for co in range(Cout):
        bp, bm = b.copy(), b.copy()
        bp[co] += e
        bm[co] -= e
        assert g["g_b"][co] == pytest.approx((L(b_=bp) - L(b_=bm)) / (2 * e), rel=1e-9, abs=1e-9)
    for idx in [(0, 1, 2, 3), (1, 2, 4, 0)]:
        vp, vm = vi.copy(), vi.copy()
        vp[idx] += e
        vm[idx] -= e
        assert g["g_vinit"][idx] == pytest.approx((L(vi_=vp) - L(vi_=vm)) / (2 * e), rel=1e-9, abs=1e-9)
    for idx in [(0, 0, 0, 0, 0), (T - 1, 1, 1, 4, 5), (K, 0, 1, 2, 3)]:
        Xp, Xm = X.copy(), X.copy()
        Xp[idx] += e
        Xm[idx] -= e
        assert g["g_in"][idx] == pytest.approx((L(X_=Xp) - L(X_=Xm)) / (2 * e), rel=1e-8, abs=1e-9)
    if alpha is not None:
        for j in range(K):
            ap, am = alpha.copy(), alpha.copy()
            ap[j] += e
            am[j] -= e
            assert g["g_alpha"][j] == pytest.approx((L(a_=ap) - L(a_=am)) / (2 * e), rel=1e-9, abs=1e-9)


# --- independent torch reference --------------------------------------------------
def _primitive(kind, a, u):
    if kind == "fast_sigmoid":
        return u / (1.0 + a * u.abs())
    return torch.atan(torch.pi / 2 * a * u) / torch.pi


class _Spike(torch.autograd.Function):
    @staticmethod
    def forward(ctx, u, kind, a):
        ctx.save_for_backward(u)
        ctx.kind, ctx.a = kind, a
        return (u >= 0).to(u.dtype)

    @staticmethod
    def backward(ctx, g):
        (u,) = ctx.saved_tensors
        with torch.enable_grad():
            x = u.detach().requires_grad_(True)
            (h,) = torch.autograd.grad(_primitive(ctx.kind, ctx.a, x).sum(), x)
        return g * h, None, None


def _torch_layer(S, W, b, *, K, mode, beta, v_th, pad, kind, a, detach, v_init, alpha):
    T = S.shape[0]
    if mode == "dense":
        K = 1
    G, ns = T // K, (K if mode == "tactp" else 1)
    decay = beta ** K if mode == "tac" else beta
    coef = alpha if (alpha is not None and mode != "dense") else [beta ** (K - 1 - j) for j in range(K)]
    U, outs = v_init, []
    for k in range(G):
        A = sum(coef[j] * S[k * K + j] for j in range(K))
        Y = F.conv2d(A, W, b, padding=pad)
        for _ in range(ns):
            V = decay * U + Y
            s = _Spike.apply(V - v_th, kind, a)
            U = V - v_th * (s.detach() if detach else s)
            outs.append(s)
    return torch.stack(outs), U


@pytest.mark.parametrize("alpha_on", [False, True])
@pytest.mark.parametrize("detach", [True, False])
@pytest.mark.parametrize("kind,a", [("fast_sigmoid", 25.0), ("arctan", 2.0)])
@pytest.mark.parametrize("mode,K", [("dense", 1), ("tac", 2), ("tactp", 2), ("tac", 4)])
def test_backward_matches_torch_autograd(oracle_mod, mode, K, kind, a, detach, alpha_on):
    O = oracle_mod
    if alpha_on and mode == "dense":
        pytest.skip("no aggregation in dense mode")
    rng = np.random.default_rng(zlib.crc32(f"{mode}{K}{kind}{detach}{alpha_on}".encode()))
    T, B, Cin, H, W, Cout = 8, 2, 2, 6, 5, 3
    S = (rng.random((T, B, Cin, H, W)) < 0.4).astype(np.uint8)
    Wt = (rng.standard_normal((Cout, Cin, 3, 3)) * 0.9).astype(np.float32)
    b = (rng.uniform(-0.1, 0.1, Cout)).astype(np.float32)
    alpha = rng.uniform(0.2, 1.0, K).astype(np.float32) if alpha_on else None
    vi = rng.uniform(-0.5, 0.5, (B, Cout, H, W))
    beta = 0.75
    T_out = T // K if mode == "tac" else T
    g_out = rng.standard_normal((T_out, B, Cout, H, W))
    g_vf = rng.standard_normal((B, Cout, H, W))

    St = torch.tensor(S, dtype=torch.float64, requires_grad=True)
    Wtt = torch.tensor(Wt, dtype=torch.float64, requires_grad=True)
    bt = torch.tensor(b, dtype=torch.float64, requires_grad=True)
    vt = torch.tensor(vi, requires_grad=True)
    at = torch.tensor(alpha, dtype=torch.float64, requires_grad=True) if alpha_on else None
    out, U = _torch_layer(St, Wtt, bt, K=K, mode=mode, beta=float(np.float32(beta)), v_th=1.0, pad=1,
                          kind=kind, a=a, detach=detach, v_init=vt,
                          alpha=None if at is None else list(at.unbind()))
    assert 0.02 < float(out.detach().mean()) < 0.95
    loss = (torch.tensor(g_out) * out).sum() + (torch.tensor(g_vf) * U).sum()
    loss.backward()
    r = O.backward(S, Wt, b, g_out, K=K, mode=mode, beta=beta, v_th=1.0, pad=1, surrogate=kind,
                   sg_alpha=a, detach_reset=detach, v_init=vi, g_vfinal=g_vf, alpha=alpha,
                   replay=out.detach().numpy().astype(np.uint8), band=1e-9)
    tol = dict(rtol=1e-9, atol=1e-10)
    np.testing.assert_allclose(r["g_W"], Wtt.grad.numpy(), **tol)
    np.testing.assert_allclose(r["g_b"], bt.grad.numpy(), **tol)
    np.testing.assert_allclose(r["g_vinit"], vt.grad.numpy(), **tol)
    np.testing.assert_allclose(r["g_in"], St.grad.numpy(), **tol)
    if alpha_on:
        np.testing.assert_allclose(r["g_alpha"], at.grad.numpy(), **tol)
