"""Pins for the CPU oracle (oracle/): each test ties the oracle to something
other than itself -- a value the paper or SPEC prints (tests/golden/), a closed
form, an invariant, a library routine (torch conv2d / max_pool2d, numpy
packbits), or the paper's own error bound evaluated exactly by enumeration.

Citations "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n.
"""
import itertools
import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

HERE = os.path.dirname(os.path.abspath(__file__))
RESETS = ["subtract", "delayed", "hard"]


def _rand_spikes(rng, shape, rho):
    return (rng.random(shape) < rho).astype(np.uint8)


def _rand_w(rng, cout, cin, r=3, s=3, gain=1.0):
    return (rng.standard_normal((cout, cin, r, s)) * gain / np.sqrt(cin * r * s)).astype(np.float32)


# --- golden hand-derived cases (Alg. 1/2, Eq. 1) -----------------------
with open(os.path.join(HERE, "golden", "lif_scalar_cases.json")) as f:
    GOLDEN = json.load(f)["cases"]


@pytest.mark.parametrize("case", GOLDEN, ids=[c["name"] for c in GOLDEN])
def test_golden_scalar_cases(oracle_mod, case):
    if "X" in case:   # continuous-valued input frames (fp64 oracle path)
        T = len(case["X"])
        S = np.array(case["X"], np.float64).reshape(T, 1, 1, 1, 1)
    else:
        T = len(case["S"])
        S = np.array(case["S"], np.uint8).reshape(T, 1, 1, 1, 1)
    W = np.full((1, 1, 1, 1), case["w"], np.float32)
    bias = None if case["bias"] is None else np.array([case["bias"]], np.float32)
    r = oracle_mod.forward(S, W, bias, K=case["K"], mode=case["mode"], beta=case["beta"],
                           v_th=case["v_th"], v_reset=case.get("v_reset", 0.0),
                           reset=case["reset"], pad=0, partial=case.get("partial", False),
                           alpha=case.get("alpha"))
    assert r["out"].ravel().tolist() == case["out"]
    assert r["v_final"].ravel()[0] == pytest.approx(case["v_final"], abs=1e-12)
    assert int(r["counts"].sum()) == sum(case["out"])


# --- conv: library routine (P5) and linearity (P4) ---------------------------
@pytest.mark.parametrize("pad,stride", [(0, 1), (1, 1), (1, 2), (2, 1)])
def test_conv_matches_torch_conv2d(oracle_mod, pad, stride):
    """Direct-loop conv == torch.nn.functional.conv2d (cross-correlation, zero
    padding) in fp64.  Catches transposed/flipped kernels, pad offsets."""
    rng = np.random.default_rng(0)
    X = rng.standard_normal((2, 3, 7, 6))
    W = _rand_w(rng, 4, 3, 3, 3)
    W[:, :, 0, 2] += 0.5          # break symmetry so a flipped kernel fails
    b = rng.standard_normal(4).astype(np.float32)
    Y = oracle_mod.conv2d(X, W, b, stride=stride, pad=pad)
    ref = F.conv2d(torch.from_numpy(X), torch.from_numpy(W.astype(np.float64)),
                   torch.from_numpy(b.astype(np.float64)), stride=stride, padding=pad).numpy()
    np.testing.assert_allclose(Y, ref, rtol=0, atol=1e-12)


def test_conv_linearity(oracle_mod):
    """W*(sum a_i X_i) = sum a_i (W*X_i), with K=4 binary frames
    weighted beta^{3-j} (Alg. 1 l.3)."""
    rng = np.random.default_rng(1)
    beta = 0.9
    Xs = [_rand_spikes(rng, (2, 3, 9, 9), 0.2).astype(np.float64) for _ in range(4)]
    W = _rand_w(rng, 5, 3)
    coeffs = [beta ** (3 - j) for j in range(4)]
    lhs = oracle_mod.conv2d(sum(c * x for c, x in zip(coeffs, Xs)), W, None, pad=1)
    rhs = sum(c * oracle_mod.conv2d(x, W, None, pad=1) for c, x in zip(coeffs, Xs))
    assert np.max(np.abs(lhs - rhs)) <= 1e-12


# --- K = 1 degeneracy (P1) ---------------------------
@pytest.mark.parametrize("reset", RESETS)
def test_k1_tac_tactp_dense_identical(oracle_mod, reset):
    rng = np.random.default_rng(2)
    S = _rand_spikes(rng, (6, 3, 2, 8, 8), 0.3)
    W = _rand_w(rng, 4, 2, gain=2.0)
    b = (rng.random(4) * 0.2 - 0.1).astype(np.float32)
    kw = dict(beta=0.8, v_th=1.0, v_reset=-0.1, reset=reset, pad=1)
    d = oracle_mod.forward(S, W, b, K=1, mode="dense", **kw)
    t = oracle_mod.forward(S, W, b, K=1, mode="tac", **kw)
    p = oracle_mod.forward(S, W, b, K=1, mode="tactp", **kw)
    assert d["out"].sum() > 0
    for r in (t, p):
        assert np.array_equal(r["out"], d["out"])
        assert np.array_equal(r["v_final"], d["v_final"])
        assert np.array_equal(r["counts"], d["counts"])


# --- no-spike regime: closed forms (P2, P3) -----------------------------------
def _torch_conv_frames(S, W):
    """conv of every frame via torch (library routine), fp64: [T,B,Cout,Ho,Wo]."""
    T, B = S.shape[:2]
    x = torch.from_numpy(S.astype(np.float64).reshape(T * B, *S.shape[2:]))
    y = F.conv2d(x, torch.from_numpy(W.astype(np.float64)), padding=1).numpy()
    return y.reshape(T, B, *y.shape[1:])


@pytest.mark.parametrize("K", [2, 4])
def test_no_spike_tac_equals_dense_at_group_ends(oracle_mod, K):
    """With v_th huge and bias 0 no neuron fires; then by linearity (App. A
    'vanishes exactly' P:457) V^TAC after group k equals the dense membrane at
    t = kK+K-1, which is the linear filter sum_{tau<=t} beta^{t-tau} W*S_tau."""
    rng = np.random.default_rng(3)
    beta = 0.9
    b32 = float(np.float32(beta))
    T = 8
    S = _rand_spikes(rng, (T, 2, 2, 6, 6), 0.3)
    W = _rand_w(rng, 3, 2, gain=2.0)
    Yt = _torch_conv_frames(S, W)
    for G in range(1, T // K + 1):
        t_end = G * K - 1
        closed = sum(b32 ** (t_end - tau) * Yt[tau] for tau in range(t_end + 1))
        r_tac = oracle_mod.forward(S[:G * K], W, None, K=K, mode="tac", beta=beta, v_th=1e30, pad=1)
        r_den = oracle_mod.forward(S[:G * K], W, None, mode="dense", beta=beta, v_th=1e30, pad=1)
        assert r_tac["out"].sum() == 0
        np.testing.assert_allclose(r_tac["v_final"], closed, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(r_den["v_final"], closed, rtol=1e-12, atol=1e-12)


def test_no_spike_tactp_closed_form(oracle_mod):
    """Alg. 2 l.5-6 with no spikes: V_{kK+K-1} = beta^K V_{kK-1} + Y_k (1-beta^K)/(1-beta),
    Y_k = W*A_k, A_k = sum_j beta^{K-1-j} S_{kK+j}."""
    rng = np.random.default_rng(4)
    beta, K, T = 0.5, 4, 12
    b32 = float(np.float32(beta))
    S = _rand_spikes(rng, (T, 2, 3, 5, 5), 0.4)
    W = _rand_w(rng, 2, 3, gain=2.0)
    Yt = _torch_conv_frames(S, W)
    V = np.zeros_like(Yt[0])
    for k in range(T // K):
        Yk = sum(b32 ** (K - 1 - j) * Yt[k * K + j] for j in range(K))   # linearity
        V = b32 ** K * V + Yk * (1 - b32 ** K) / (1 - b32)
    r = oracle_mod.forward(S, W, None, K=K, mode="tactp", beta=beta, v_th=1e30, pad=1)
    np.testing.assert_allclose(r["v_final"], V, rtol=1e-12, atol=1e-12)


# --- zero input (P7) ----------------------------------------------------
@pytest.mark.parametrize("reset", RESETS)
@pytest.mark.parametrize("mode", ["dense", "tac", "tactp"])
def test_zero_input_no_spikes(oracle_mod, mode, reset):
    S = np.zeros((4, 2, 1, 5, 5), np.uint8)
    W = _rand_w(np.random.default_rng(5), 3, 1, gain=5.0)
    r = oracle_mod.forward(S, W, None, K=2, mode=mode, beta=0.9, reset=reset, pad=1)
    assert r["out"].sum() == 0 and np.all(r["v_final"] == 0) and r["counts"].sum() == 0


# --- shapes and conv-call accounting (P8) -----
def test_output_steps_and_call_accounting(oracle_mod):
    S = np.zeros((16, 1, 1, 4, 4), np.uint8)
    W = np.zeros((2, 1, 3, 3), np.float32)
    assert oracle_mod.forward(S, W, K=4, mode="tac", pad=1)["out"].shape[0] == 4      # T/K
    assert oracle_mod.forward(S, W, K=4, mode="tactp", pad=1)["out"].shape[0] == 16   # T
    assert oracle_mod.forward(S, W, mode="dense", pad=1)["out"].shape[0] == 16
    # Table tab:dvsg conv-call column, 5 layers at T=16: 80 / 40 / 20 / 10
    assert oracle_mod.temporal_extents(16, [1] * 5, ["dense"] * 5)[1] == 80
    for K, calls in [(2, 40), (4, 20), (8, 10)]:
        ext, c, t_final = oracle_mod.temporal_extents(16, [K] * 5, ["tactp"] * 5)
        assert c == calls and t_final == 16                   # App. B: TAC-TP keeps T
    # App. B: cascaded TAC K=2 over 5 layers at T=16 -> 16/2^5 = 0.5 (invalid)
    with pytest.raises(ValueError):
        oracle_mod.temporal_extents(16, [2] * 5, ["tac"] * 5)
    assert oracle_mod.temporal_extents(32, [2] * 5, ["tac"] * 5)[2] == 1
    with pytest.raises(ValueError):
        oracle_mod.forward(np.zeros((6, 1, 1, 4, 4), np.uint8), W, K=4, mode="tac", pad=1)


# --- chaining with v_init / v_final (P12; reading R4/R5) ----------------------
@pytest.mark.parametrize("reset", RESETS)
@pytest.mark.parametrize("mode", ["dense", "tac", "tactp"])
def test_chaining_v_init_v_final(oracle_mod, mode, reset):
    rng = np.random.default_rng(6)
    S = _rand_spikes(rng, (8, 2, 2, 6, 6), 0.3)
    W = _rand_w(rng, 3, 2, gain=2.5)
    b = (rng.random(3) * 0.2 - 0.1).astype(np.float32)
    kw = dict(K=2, mode=mode, beta=0.7, v_th=1.0, v_reset=0.1, reset=reset, pad=1)
    full = oracle_mod.forward(S, W, b, **kw)
    a = oracle_mod.forward(S[:4], W, b, **kw)
    c = oracle_mod.forward(S[4:], W, b, v_init=a["v_final"], **kw)
    assert np.array_equal(np.concatenate([a["out"], c["out"]]), full["out"])
    assert np.array_equal(c["v_final"], full["v_final"])
    assert full["out"].sum() > 0


# --- Theorem 1, exact expectation by enumeration (P10) ---
def _thm1_error(O, rho, w, K, reset, T=8, beta=0.9):
    allS = np.array(list(itertools.product([0, 1], repeat=T)), np.uint8)
    Sx = np.ascontiguousarray(allS.T.reshape(T, len(allS), 1, 1, 1))
    W = np.full((1, 1, 1, 1), w, np.float32)
    d = O.forward(Sx, W, mode="dense", beta=beta, reset=reset)
    t = O.forward(Sx, W, K=K, mode="tac", beta=beta, reset=reset)
    n = allS.sum(1)
    p = rho ** n * (1 - rho) ** (T - n)
    err = float((p * (d["v_final"].ravel() - t["v_final"].ravel()) ** 2).sum())
    b32 = float(np.float32(beta))
    # C = V_th^2 N_spatial / (1 - beta^{2K}), N_spatial = 1, ||W||_F^2 = w^2
    bound = 1.0 / (1 - b32 ** (2 * K)) * rho * (1 - rho) * K * w * w
    return err, bound


@pytest.mark.parametrize("reset", ["subtract", "delayed"])
def test_theorem1_bound_holds_at_paper_rate(oracle_mod, reset):
    """E||V_T^exact - V_T^TAC||^2 <= C rho(1-rho) K ||W||_F^2 evaluated EXACTLY over
    all 2^8 inputs of a scalar neuron at the paper's firing rate rho=0.1."""
    for w in (0.25, 0.5, 1.0, 1.5):
        prev = -1.0
        for K in (2, 4, 8):
            err, bound = _thm1_error(oracle_mod, 0.1, w, K, reset)
            assert err <= bound, (w, K, err, bound)
            if reset == "subtract":
                assert err >= prev - 1e-15      # monotone in K for SUBTRACT
                prev = err


def test_theorem1_bound_is_not_general(oracle_mod):
    """Reading D10: the bound is garbled and fails at rho=0.5, w=1.5,
    K=4 -- recorded so the bound is never used as a GPU assertion."""
    err, bound = _thm1_error(oracle_mod, 0.5, 1.5, 4, "subtract")
    assert err > bound


# --- LIF invariants ------------------------------------------------
def test_monotone_drive_scalar(oracle_mod):
    """Subtract reset, non-negative inputs: raising the input at one step never
    lowers the spike count, exhaustive over a small grid."""
    T = 5
    levels = [0.0, 0.25, 0.5, 0.75, 1.0, 1.25]
    seqs = np.array(list(itertools.product(levels, repeat=T)))
    # input I_t = W*S_t with C_in = T one-hot channels (S_t hits channel t only)
    # and a 1x1 weight vector holding the input sequence.
    S = np.zeros((T, 1, T, 1, 1), np.uint8)
    for t in range(T):
        S[t, :, t] = 1
    res = {}
    for seq in seqs:
        W = seq.astype(np.float32).reshape(1, T, 1, 1)
        r = oracle_mod.forward(S, W, mode="dense", beta=0.5, reset="subtract")
        res[tuple(seq)] = int(r["out"].sum())
    for seq, c in res.items():
        for t in range(T):
            li = levels.index(seq[t])
            if li + 1 < len(levels):
                up = list(seq)
                up[t] = levels[li + 1]
                assert res[tuple(up)] >= c


def test_boundedness(oracle_mod):
    """|input| <= M  =>  V after reset <= M/(1-beta) + v_th."""
    rng = np.random.default_rng(7)
    S = _rand_spikes(rng, (20, 4, 3, 6, 6), 0.5)
    W = _rand_w(rng, 4, 3, gain=4.0)
    beta = 0.9
    M = float(np.abs(W).sum(axis=(1, 2, 3)).max())
    for mode, K in (("dense", 1), ("tactp", 4), ("tac", 4)):
        r = oracle_mod.forward(S, W, K=K, mode=mode, beta=beta, pad=1)
        Meff = M * (sum(beta ** j for j in range(K)) if mode != "dense" else 1.0)
        assert np.all(r["v_final"] <= Meff / (1 - beta) + 1.0)


# --- replay protocol -----------------------------------------------------------
def test_replay_protocol(oracle_mod):
    rng = np.random.default_rng(8)
    S = _rand_spikes(rng, (8, 2, 2, 6, 6), 0.3)
    W = _rand_w(rng, 3, 2, gain=2.5)
    kw = dict(K=2, mode="tactp", beta=0.5, pad=1)
    ref = oracle_mod.forward(S, W, **kw)
    same = oracle_mod.forward(S, W, replay=ref["out"], **kw)
    assert same["mismatch"] == 0 and np.array_equal(same["v_final"], ref["v_final"])
    bad = ref["out"].copy()
    idx = np.argwhere(bad == 1)[0]
    bad[tuple(idx)] = 0
    r = oracle_mod.forward(S, W, replay=bad, **kw)
    assert r["mismatch"] >= 1
    # a huge band excuses every decision and follows the replayed spikes exactly
    r2 = oracle_mod.forward(S, W, replay=bad, band=1e9, **kw)
    assert r2["mismatch"] == 0 and r2["excused"] == bad.size
    assert np.array_equal(r2["out"], bad)


# --- OR-pool and packed format --------------------------------------------------
def test_or_pool_matches_max_pool(oracle_mod):
    rng = np.random.default_rng(9)
    x = _rand_spikes(rng, (3, 2, 4, 8, 6), 0.2)
    ref = F.max_pool2d(torch.from_numpy(x.reshape(6, 4, 8, 6)).float(), 2).numpy()
    assert np.array_equal(oracle_mod.or_pool2(x).reshape(6, 4, 4, 3), ref.astype(np.uint8))


def test_pack_hand_example(oracle_mod):
    """include/tacsnn.h layout: bit (c, x) of a row sits at r = x*C + c, LSB first."""
    d = np.zeros((1, 1, 2, 1, 3), np.uint8)   # T=1,B=1,C=2,H=1,W=3
    d[0, 0, 1, 0, 2] = 1                      # c=1, x=2 -> r=5
    d[0, 0, 0, 0, 0] = 1                      # c=0, x=0 -> r=0
    p = oracle_mod.pack_spikes(d)
    assert p.shape == (1, 1, 1, 1) and int(p[0, 0, 0, 0]) == (1 << 5) | 1
    d2 = np.zeros((1, 1, 1, 1, 40), np.uint8)
    d2[0, 0, 0, 0, 33] = 1                    # second word, bit 1
    p2 = oracle_mod.pack_spikes(d2)
    assert p2.shape[-1] == 2 and int(p2[0, 0, 0, 0]) == 0 and int(p2[0, 0, 0, 1]) == 2


@pytest.mark.parametrize("C,W", [(1, 28), (2, 128), (32, 13), (128, 8), (8, 26), (3, 5)])
def test_pack_roundtrip(oracle_mod, C, W):
    rng = np.random.default_rng(C * 1000 + W)
    d = _rand_spikes(rng, (3, 2, C, 4, W), 0.3)
    p = oracle_mod.pack_spikes(d)
    assert p.shape == (3, 2, 4, (W * C + 31) // 32)
    assert np.array_equal(oracle_mod.unpack_spikes(p, C, W), d)


# --- continuous-valued input ------------------------
@pytest.mark.parametrize("mode", ["dense", "tac", "tactp"])
def test_real_input_path_equals_spike_path_on_binary_frames(oracle_mod, mode):
    """{0,1} frames given as floats follow the same arithmetic as u8 spikes: bitwise."""
    rng = np.random.default_rng(31)
    S = (rng.random((8, 2, 2, 9, 9)) < 0.3).astype(np.uint8)
    W = _rand_w(rng, 4, 2, gain=2.0)
    b = (rng.standard_normal(4) * 0.1).astype(np.float32)
    r1 = oracle_mod.forward(S, W, b, K=4, mode=mode, beta=0.9, pad=1)
    r2 = oracle_mod.forward(S.astype(np.float64), W, b, K=4, mode=mode, beta=0.9, pad=1)
    assert np.array_equal(r1["out"], r2["out"]) and np.array_equal(r1["v_final"], r2["v_final"])


@pytest.mark.parametrize("K", [2, 4])
def test_real_input_no_spike_tac_equals_dense(oracle_mod, K):
    """Linearity holds for continuous input too: with no spikes and no bias,
    V^TAC after group k equals V^dense at t = kK + K - 1."""
    rng = np.random.default_rng(32)
    X = rng.gamma(1.0, 0.5, (8, 2, 2, 7, 7))
    W = _rand_w(rng, 3, 2)
    for k in range(8 // K):
        T = (k + 1) * K
        d = oracle_mod.forward(X[:T], W, None, K=1, mode="dense", beta=0.9, v_th=1e30, pad=1)
        t = oracle_mod.forward(X[:T], W, None, K=K, mode="tac", beta=0.9, v_th=1e30, pad=1)
        np.testing.assert_allclose(t["v_final"], d["v_final"], rtol=1e-12, atol=1e-12)


def test_theorem1_statistical_c1_shape(oracle_mod):
    """P11: the literal Theorem 1 bound at a C1-like shape (Bernoulli
    rho=0.1 inputs, beta=0.9, T=16, 1->8 channels 3x3 on 28x28, pad 0, 40 samples):
    E||V^dense_T - V^TAC_T||^2 <= V_th^2 N / (1 - beta^{2K}) * rho (1-rho) K ||W||_F^2
    (N = output pixels) holds, with the error growing in K."""
    rng = np.random.default_rng(40)
    T, B, rho = 16, 40, 0.1
    S = _rand_spikes(rng, (T, B, 1, 28, 28), rho)
    W = _rand_w(rng, 8, 1, gain=1.0)
    d = oracle_mod.forward(S, W, K=1, mode="dense", beta=0.9)
    b32 = float(np.float32(0.9))
    prev = -1.0
    for K in (2, 4, 8):
        t = oracle_mod.forward(S, W, K=K, mode="tac", beta=0.9)
        err = float(((d["v_final"] - t["v_final"]) ** 2).sum(axis=(1, 2, 3)).mean())
        n_spatial = 26 * 26
        bound = n_spatial / (1 - b32 ** (2 * K)) * rho * (1 - rho) * K * float((W.astype(np.float64) ** 2).sum())
        assert err <= bound, (K, err, bound)
        assert err > prev, (K, err, prev)
        prev = err


# --- partial last group (K does not divide T, reading D6') -----
@pytest.mark.parametrize("reset", RESETS)
@pytest.mark.parametrize("mode", ["tac", "tactp"])
def test_partial_last_group_is_a_short_group(oracle_mod, mode, reset):
    """With partial=True and T = (G-1) K + K', the layer equals the first (G-1) K frames
    with group size K followed, through v_init = v_final, by the last K' frames as one
    group of size K' (A, decay beta^K' and step count all of the short group)."""
    rng = np.random.default_rng(50)
    S = _rand_spikes(rng, (10, 2, 2, 6, 6), 0.3)
    W = _rand_w(rng, 3, 2, gain=2.5)
    b = (rng.random(3) * 0.2 - 0.1).astype(np.float32)
    kw = dict(mode=mode, beta=0.8, v_th=1.0, v_reset=0.1, reset=reset, pad=1)
    full = oracle_mod.forward(S, W, b, K=4, partial=True, **kw)
    a = oracle_mod.forward(S[:8], W, b, K=4, **kw)
    c = oracle_mod.forward(S[8:], W, b, K=2, v_init=a["v_final"], **kw)
    assert np.array_equal(np.concatenate([a["out"], c["out"]]), full["out"])
    assert np.array_equal(c["v_final"], full["v_final"])
    assert full["out"].shape[0] == (3 if mode == "tac" else 10)


def test_partial_groups_paper_T25(oracle_mod):
    """The paper's T = 25 with K = 4 / 8 / 16: a TAC layer emits
    ceil(25/K) = 7 / 4 / 2 steps (one per conv call) instead of 25."""
    rng = np.random.default_rng(51)
    S = _rand_spikes(rng, (25, 1, 1, 5, 5), 0.2)
    W = _rand_w(rng, 2, 1)
    steps = [oracle_mod.forward(S, W, K=K, mode="tac", partial=True, pad=1)["out"].shape[0]
             for K in (4, 8, 16)]
    assert steps == [7, 4, 2]
    with pytest.raises(ValueError):
        oracle_mod.forward(S, W, K=4, mode="tac", pad=1)   # K must divide T without partial


# --- P9: exhaustive batch, oracle vs an independent brute force ---------------
def _exhaustive_inputs():
    """Every binary input of a 1-channel 2x2 image over T = 4 steps: [4, 65536, 1, 2, 2]."""
    bits = np.array(list(itertools.product([0, 1], repeat=16)), np.uint8)
    return np.ascontiguousarray(bits.reshape(-1, 4, 1, 2, 2).transpose(1, 0, 2, 3, 4))


@pytest.mark.parametrize("reset", RESETS)
@pytest.mark.parametrize("mode", ["dense", "tac", "tactp"])
def test_exhaustive_batch_bruteforce(oracle_mod, mode, reset):
    """SURVEY P9 on CPU: all 2^16 inputs in one batch; binary-exact weights, bias, beta and
    v_reset make every value exact in fp64, so the C oracle and the brute force
    (tests/bruteforce.py: loops straight from Eq. (1) / Alg. 1 / Alg. 2) must agree bitwise."""
    import bruteforce
    S = _exhaustive_inputs()
    rng = np.random.default_rng(9)
    W = (rng.integers(-24, 25, (4, 1, 3, 3)) / 16.0).astype(np.float32)
    b = (rng.integers(-2, 3, 4) / 16.0).astype(np.float32)
    kw = dict(K=2, mode=mode, beta=0.5, v_th=1.0, reset=reset, v_reset=-0.25)
    r = oracle_mod.forward(S, W, b, pad=1, **kw)
    out, V = bruteforce.layer(S, W, b, pad=1, **kw)
    assert 0.02 < out.mean() < 0.98
    assert np.array_equal(r["out"], out)
    assert np.array_equal(r["v_final"], V)
    assert np.array_equal(r["counts"], out.sum(axis=(0, 3, 4)))


@pytest.mark.parametrize("mode", ["tac", "tactp"])
def test_agg_weights_equal_default_when_alpha_is_beta_powers(oracle_mod, mode):
    """alpha_j = beta^{K-1-j} (binary-exact at beta = 1/2) reproduces the default
    aggregation bitwise; alpha scaled by 2 with W halved is the same layer (linearity)."""
    rng = np.random.default_rng(4)
    S = _rand_spikes(rng, (6, 2, 2, 7, 7), 0.3)
    W = (rng.integers(-24, 25, (3, 2, 3, 3)) / 32.0).astype(np.float32)
    kw = dict(K=3, mode=mode, beta=0.5, v_th=1.0, pad=1)
    d = oracle_mod.forward(S, W, None, **kw)
    a = oracle_mod.forward(S, W, None, alpha=[0.25, 0.5, 1.0], **kw)
    h = oracle_mod.forward(S, W / 2, None, alpha=[0.5, 1.0, 2.0], **kw)
    assert d["out"].sum() > 0
    for r in (a, h):
        assert np.array_equal(r["out"], d["out"]) and np.array_equal(r["v_final"], d["v_final"])
    o = oracle_mod.forward(S, W, None, alpha=[1.0, 0.5, 0.25], **kw)   # reversed: a different layer
    assert not np.array_equal(o["v_final"], d["v_final"])


def test_vote_pin():
    """VotingLayer by hand: 2 classes x 3 voters, T_out = 4: class
    scores are the voters' mean firing rates, (1 + 2 + 3) / 12 and (0 + 4 + 4) / 12."""
    from oracle import oracle as O
    s = O.vote(np.array([[1, 2, 3, 0, 4, 4]]), 3, 4)
    assert s.shape == (1, 2)
    assert s[0, 0] == 0.5 and abs(s[0, 1] - 8 / 12) < 1e-15
