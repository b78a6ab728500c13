"""GPU parity of the training path: tac_conv_lif_forward_train +
tac_conv_lif_backward through the C ABI against the oracle's fp64 BPTT
(oracle.backward, pinned in tests/test_oracle_backward.py), on the device's own
spike trajectory (replay, band 1e-3 v_th), plus the OR-pool and its MaxPool2d
backward.

Tolerance (reading R12): every gradient tensor within
tol = 1e-3 + 2 alpha 2e-4 of its own max |value| elementwise (fast sigmoid alpha 25:
1.1e-2; arctan alpha 2: 1.8e-3).  The device's conv operands carry up to ~1.6e-5
max|w| weight error (two int8 slices; fp16 hi + lo is ~2^-22), which moves V by up
to ~1e-4, and the surrogate amplifies a V error into the gradient by its slope
|h'| <= 2 alpha; fp32 batch sums add ~1e-6.
"""
import zlib

import numpy as np
import pytest
import torch

import _parity as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_13810_b200 import build, tacsnn
    build.build()
    return tacsnn


@pytest.fixture(scope="module")
def O():
    from oracle import oracle
    oracle.build()
    return oracle


def _tol(alpha):
    return 1e-3 + 2.0 * alpha * 2e-4


def _close(dev, ref, label, rel=2e-3):
    dev = np.asarray(dev, np.float64)
    scale = max(np.abs(ref).max(), 1e-30)
    err = np.abs(dev - ref).max()
    assert err <= rel * scale, f"{label}: max err {err:.3e} vs scale {scale:.3e} (ratio {err / scale:.2e})"
    return err / scale


def _cl_to_oracle(a):   # [T,B,H,W,C] -> [T,B,C,H,W]
    return np.ascontiguousarray(np.asarray(a).transpose(0, 1, 4, 2, 3))


CASES = [
    # name, (T,B,Cin,H,W,Cout,pad), beta, gain, rho
    ("mnistL1", (8, 3, 1, 28, 28, 32, 0), 0.9, 2.5, 0.15),
    ("dvsL1", (8, 2, 2, 32, 32, 128, 1), 0.5, 6.0, 0.08),
    ("mnistL2", (8, 3, 32, 13, 13, 64, 0), 0.9, 3.0, 0.15),
    ("dvsL2", (8, 2, 128, 16, 16, 128, 1), 0.5, 3.0, 0.1),
    # fully connected layers (1x1 conv of a 1x1 image; backward = two tiled GEMMs)
    ("fc1600", (8, 5, 1600, 1, 1, 128, 0, 1), 0.9, 3.0, 0.15),
    ("fc512", (8, 3, 512, 1, 1, 110, 0, 1), 0.5, 4.0, 0.1),
]


@pytest.mark.parametrize("engine", ["simt", "tcgen05"])
@pytest.mark.parametrize("mode,K", [("dense", 1), ("tac", 4), ("tactp", 2), ("tactp", 4)])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_layer_backward_parity(T, O, case, mode, K, engine):
    name, shape, beta, gain, rho = case
    Tn, B, Cin, H, W, Cout, pad = shape[:7]
    R = shape[7] if len(shape) > 7 else 3
    spec = T.LayerSpec(T=Tn, B=B, C_in=Cin, H=H, W=W, C_out=Cout, R=R, S=R, pad=pad, K=K, mode=mode, beta=beta,
                       out_pool=1, engine=engine)
    try:
        assert spec.engine_used() == engine
    except RuntimeError:
        pytest.skip("outside the engine's envelope")
    kind, a, detach = ("fast_sigmoid", 25.0, False) if beta == 0.9 else ("arctan", 2.0, True)
    seed = zlib.crc32(f"{name}{mode}{K}".encode())
    g = torch.Generator().manual_seed(seed)
    S = (torch.rand((Tn, B, Cin, H, W), generator=g) < rho).to(torch.uint8).numpy()
    from paper_2603_13810_b200 import synth
    w, b = synth.weights(seed % 1000, Cout, Cin, R, R, gain=gain if mode != "tactp" else gain / 1.5)
    prep = T.prepare_weights(spec, w, b)
    x = T.pack(torch.from_numpy(S).cuda())
    hc, wc = spec.conv_hw
    vi = (torch.rand((B, hc, wc, Cout), generator=g) * 0.6 - 0.3).cuda()
    out, vf, _, y_seq = T.conv_lif_train(spec, prep, x, v_init=vi, want_v_final=True)
    T_out = out.shape[0]
    gs = torch.randn((T_out, B, hc, wc, Cout), generator=g).cuda()
    gvf = torch.randn((B, hc, wc, Cout), generator=g).cuda()
    r = T.conv_lif_backward(spec, prep, x, y_seq, gs, v_init=vi, g_v_final=gvf, surrogate=kind, alpha=a,
                            detach_reset=detach, want_v_init_grad=True)
    torch.cuda.synchronize()
    D = O.unpack_spikes(P.to_u32(out), Cout, wc)
    assert 0.01 < D.mean() < 0.9, D.mean()
    vi_o = vi.cpu().numpy().transpose(0, 3, 1, 2).astype(np.float64)
    # the training forward is the inference forward: spikes pass the replay parity
    fw = O.forward(S, w.numpy(), b.numpy(), K=K, mode=mode, beta=beta, pad=pad, v_init=vi_o, replay=D,
                   band=P.BAND)
    assert fw["mismatch"] == 0
    ref = O.backward(S, w.numpy(), b.numpy(), _cl_to_oracle(gs.cpu().numpy()), K=K, mode=mode, beta=beta,
                     pad=pad, surrogate=kind, sg_alpha=a, detach_reset=detach, v_init=vi_o,
                     g_vfinal=gvf.cpu().numpy().transpose(0, 3, 1, 2), replay=D, band=P.BAND)
    lab = f"{name}/{mode}/K{K}/{engine}"
    tol = _tol(a)
    _close(r["g_weight"].cpu().numpy(), ref["g_W"], lab + " g_W", tol)
    _close(r["g_bias"].cpu().numpy(), ref["g_b"], lab + " g_b", tol)
    _close(_cl_to_oracle(r["g_input"].cpu().numpy()), ref["g_in"], lab + " g_in", tol)
    _close(r["g_v_init"].cpu().numpy().transpose(0, 3, 1, 2), ref["g_vinit"], lab + " g_vinit", tol)


@pytest.mark.parametrize("engine", ["simt", "tcgen05"])
def test_backward_agg_weights_and_real_input(T, O, engine):
    """Learnable alpha with dL/dalpha, on continuous-valued input frames."""
    from paper_2603_13810_b200 import synth
    Tn, B, Cin, H, W, Cout, K = 8, 2, 2, 24, 24, 64, 4
    alpha = (0.2, 0.45, 0.7, 1.0)
    spec = T.LayerSpec(T=Tn, B=B, C_in=Cin, H=H, W=W, C_out=Cout, pad=1, K=K, mode="tac", beta=0.9,
                       out_pool=1, input="real", agg_weights=alpha, engine=engine)
    assert spec.engine_used() == engine
    X = synth.dvs_log_counts(3, Tn, B, H, W)                   # [T,B,C,H,W]
    w, b = synth.weights(21, Cout, Cin, gain=3.0)
    prep = T.prepare_weights(spec, w, b)
    x = X.permute(0, 1, 3, 4, 2).contiguous().cuda()
    out, _, _, y_seq = T.conv_lif_train(spec, prep, x)
    g = torch.Generator().manual_seed(5)
    gs = torch.randn((out.shape[0], B, H, W, Cout), generator=g).cuda()
    r = T.conv_lif_backward(spec, prep, x, y_seq, gs, surrogate="fast_sigmoid", alpha=25.0, want_agg_grad=True)
    torch.cuda.synchronize()
    D = O.unpack_spikes(P.to_u32(out), Cout, W)
    assert 0.01 < D.mean() < 0.9
    ref = O.backward(X.numpy().astype(np.float64), w.numpy(), b.numpy(), _cl_to_oracle(gs.cpu().numpy()), K=K,
                     mode="tac", beta=0.9, pad=1, surrogate="fast_sigmoid", sg_alpha=25.0, alpha=alpha,
                     replay=D, band=P.BAND)
    tol = _tol(25.0)
    _close(r["g_weight"].cpu().numpy(), ref["g_W"], "alpha g_W", tol)
    _close(r["g_bias"].cpu().numpy(), ref["g_b"], "alpha g_b", tol)
    _close(_cl_to_oracle(r["g_input"].cpu().numpy()), ref["g_in"], "alpha g_in", tol)
    _close(r["g_agg_weights"].cpu().numpy(), ref["g_alpha"], "g_alpha", tol)


@pytest.mark.parametrize("C,H,W", [(32, 26, 26), (128, 16, 16), (3, 11, 13), (32, 11, 13), (64, 7, 6)])
def test_or_pool2_and_backward(T, O, C, H, W):
    g = torch.Generator().manual_seed(C + H)
    S = (torch.rand((3, 2, C, H, W), generator=g) < 0.3).to(torch.uint8)
    x = T.pack(S.cuda())
    pooled = T.or_pool2(x, C, W)
    torch.cuda.synchronize()
    assert np.array_equal(O.unpack_spikes(P.to_u32(pooled), C, W // 2), O.or_pool2(S.numpy()))
    # backward against torch's MaxPool2d autograd (CPU, fp64) on the same binary maps
    gp = torch.randn((3, 2, H // 2, W // 2, C), generator=g, dtype=torch.float64)
    xs = S.to(torch.float64).reshape(6, C, H, W).requires_grad_(True)
    y = torch.nn.functional.max_pool2d(xs, 2)
    y.backward(gp.reshape(6, H // 2, W // 2, C).permute(0, 3, 1, 2))
    ref = xs.grad.reshape(3, 2, C, H, W).permute(0, 1, 3, 4, 2).numpy()
    dev = T.or_pool2_backward(x, gp.float().cuda(), C, W)
    torch.cuda.synchronize()
    np.testing.assert_allclose(dev.cpu().numpy(), ref, rtol=1e-6, atol=1e-6)


def test_two_layer_stack_backward(T, O):
    """conv1 (1->32, 28x28) -> OR-pool -> conv2 (32->64): the pooled layer's input gradient
    flows through tac_or_pool2_backward into layer 1's backward; every stage against the
    oracle / torch composition on the device's spikes."""
    from paper_2603_13810_b200 import configs
    cfg = configs.CONFIGS["C2"]
    specs = [s.replace(out_pool=1) for s in configs.layer_plan(cfg, mode="tac", K=4, B=4)]
    (w1, b1), (w2, b2) = configs.layer_weights(cfg)
    S = configs.make_inputs(cfg, B=4).numpy()
    p1, p2 = T.prepare_weights(specs[0], w1, b1), T.prepare_weights(specs[1], w2, b2)
    x = T.pack(torch.from_numpy(S).cuda())
    o1, _, _, y1 = T.conv_lif_train(specs[0], p1, x)
    o1p = T.or_pool2(o1, 32, 26)
    o2, _, _, y2 = T.conv_lif_train(specs[1], p2, o1p)
    g = torch.Generator().manual_seed(8)
    g2 = torch.randn((o2.shape[0], 4, 11, 11, 64), generator=g).cuda()
    r2 = T.conv_lif_backward(specs[1], p2, o1p, y2, g2)
    g1 = T.or_pool2_backward(o1, r2["g_input"], 32, 26)
    r1 = T.conv_lif_backward(specs[0], p1, x, y1, g1, want_input_grad=False)
    torch.cuda.synchronize()
    D1 = O.unpack_spikes(P.to_u32(o1), 32, 26)
    D1p = O.unpack_spikes(P.to_u32(o1p), 32, 13)
    D2 = O.unpack_spikes(P.to_u32(o2), 64, 11)
    kw = dict(mode="tac", beta=0.9, pad=0, surrogate="fast_sigmoid", sg_alpha=25.0, band=P.BAND)
    ref2 = O.backward(D1p, w2.numpy(), b2.numpy(), _cl_to_oracle(g2.cpu().numpy()), K=specs[1].K, replay=D2, **kw)
    tol = _tol(25.0)
    _close(r2["g_weight"].cpu().numpy(), ref2["g_W"], "L2 g_W", tol)
    _close(_cl_to_oracle(r2["g_input"].cpu().numpy()), ref2["g_in"], "L2 g_in", tol)
    # pool backward in torch on the oracle's L2 input gradient
    xs = torch.from_numpy(D1.astype(np.float64)).reshape(-1, 32, 26, 26).requires_grad_(True)
    torch.nn.functional.max_pool2d(xs, 2).backward(torch.from_numpy(ref2["g_in"]).reshape(-1, 32, 13, 13))
    g1_ref = xs.grad.reshape(D1.shape).numpy()
    ref1 = O.backward(S, w1.numpy(), b1.numpy(), g1_ref, K=specs[0].K, replay=D1, want_input=False, **kw)
    _close(r1["g_weight"].cpu().numpy(), ref1["g_W"], "L1 g_W", tol)
    _close(r1["g_bias"].cpu().numpy(), ref1["g_b"], "L1 g_b", tol)


@pytest.mark.parametrize("cfg_name,mode,K", [("C2", "tac", 4), ("C2", "dense", 1), ("C4", "tactp", 2)])
def test_trainable_network_forward_equals_inference(T, cfg_name, mode, K):
    """TrainableNetwork: the training forward (unpooled layers + tac_or_pool2) gives bitwise
    the inference forward's final spikes and counts; the backward chain yields finite
    gradients of the right shapes for every layer."""
    from paper_2603_13810_b200 import configs, network
    cfg = configs.CONFIGS[cfg_name]
    B = 4 if cfg_name == "C2" else 1
    if cfg.inputs == "dvs":
        specs, weights = configs.layer_plan(cfg, mode=mode, K=K, B=B), configs.layer_weights(cfg)
    else:
        specs, weights = configs.network_plan(cfg, mode=mode, K=K, B=B), configs.network_weights(cfg)
    x = T.pack(configs.make_inputs(cfg, B=B, device="cuda"))
    y_inf, c_inf, _, _ = network.Network(specs, weights).forward(x)
    tnet = network.TrainableNetwork(specs, weights)
    y, cnt, tape = tnet.forward_train(x)
    assert torch.equal(y, y_inf) and torch.equal(cnt, c_inf[-1])
    s_last = tape[-1][0]
    g = torch.ones((tape[-1][4].shape[0], B, *s_last.conv_hw, s_last.C_out), device="cuda") * 0.01
    grads = tnet.backward(tape, g)
    torch.cuda.synchronize()
    for spec, r in zip(specs, grads):
        assert tuple(r["g_weight"].shape) == (spec.C_out, spec.C_in, spec.R, spec.S)
        assert torch.isfinite(r["g_weight"]).all() and torch.isfinite(r["g_bias"]).all()
    assert any(float(r["g_weight"].abs().sum()) > 0 for r in grads)
