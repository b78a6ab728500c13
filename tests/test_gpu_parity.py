"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

All inputs come from the seeded generators (paper_2603_13810_b200.synth); the
oracle and the device see identical spikes.  See tests/_parity.py for the
replay protocol and tolerances (north_star: bit-exact spikes outside a 1e-3
band around v_th, membranes within 1e-3 relative).
"""
import itertools
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


def _w(seed, cout, cin, gain, r=3, s=3):
    from paper_2603_13810_b200 import synth
    return synth.weights(seed, cout, cin, r, s, gain=gain)


def _spikes(seed, shape, rho):
    g = torch.Generator().manual_seed(seed)
    return (torch.rand(shape, generator=g) < rho).to(torch.uint8).numpy()


ENGINES = ["simt", "tcgen05"]


def _engine_or_skip(spec, engine):
    s = spec.replace(engine=engine)
    try:
        assert s.engine_used() == engine
    except RuntimeError:
        pytest.skip(f"{engine} does not take this layer")
    return s


# ---------------------------------------------------------------- formats ----
@pytest.mark.parametrize("C,H,W", [(1, 28, 28), (2, 128, 128), (32, 13, 13), (128, 8, 8),
                                   (3, 5, 7), (8, 26, 26), (1, 5, 96), (2, 7, 48)])
def test_pack_unpack_match_oracle_format(T, O, C, H, W):
    d = _spikes(C * 100 + W, (3, 2, C, H, W), 0.3)
    p = T.pack(torch.from_numpy(d).cuda())
    assert np.array_equal(P.to_u32(p), O.pack_spikes(d))
    assert np.array_equal(T.unpack(p, C, W).cpu().numpy(), d)
    assert T.last_launch_count() == 1


# ------------------------------------------------------- single layers ------
LAYER_CASES = [
    # name, (T,B,Cin,H,W,Cout,pad,pool), gain, rho
    ("C1", (8, 4, 1, 28, 28, 8, 0, 1), 2.5, 0.1),
    ("mnistL1", (8, 3, 1, 28, 28, 32, 0, 2), 2.5, 0.15),
    ("mnistL2", (8, 3, 32, 13, 13, 64, 0, 1), 3.5, 0.15),
    ("dvsL1", (4, 2, 2, 128, 128, 128, 1, 2), 7.1, 0.03),
    ("dvsL2", (4, 2, 128, 64, 64, 128, 1, 2), 3.5, 0.1),
    ("dvsL5", (8, 5, 128, 8, 8, 128, 1, 2), 3.5, 0.1),
    ("ragged", (8, 3, 3, 13, 11, 24, 1, 1), 2.0, 0.3),
    ("wide_cin", (4, 2, 96, 10, 9, 48, 1, 2), 2.5, 0.2),
    # every C_in / C_out the int8 tcgen05 envelope admits (C_in 32k <= 128, C_out 8, 16, 32k)
    ("cin64", (4, 2, 64, 12, 16, 32, 1, 2), 2.5, 0.15),
    ("cin96_cout96", (4, 2, 96, 10, 9, 96, 1, 2), 2.5, 0.2),
    ("cin64_cout128", (4, 2, 64, 9, 20, 128, 0, 1), 2.5, 0.15),
    ("cout8_int8", (4, 2, 32, 12, 12, 8, 1, 1), 2.5, 0.2),
    ("cout16_int8", (4, 3, 32, 11, 14, 16, 1, 2), 2.5, 0.2),
    ("cin128_cout96", (4, 2, 128, 8, 8, 96, 1, 2), 3.0, 0.1),
    # fp16-halo path (C_in <= 8): LDG producers (rows not 16-B multiples) and TMA
    ("rgb", (4, 2, 3, 20, 19, 32, 1, 2), 2.5, 0.2),
    ("cin6_pad0", (4, 2, 6, 9, 13, 16, 0, 1), 2.5, 0.2),
    ("cin4_tma", (4, 2, 4, 24, 32, 64, 1, 2), 2.5, 0.2),
    ("cin8_tma", (4, 2, 8, 17, 48, 128, 1, 1), 2.5, 0.2),
]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("mode,K,beta", [("tac", 2, 0.5), ("tactp", 2, 0.5), ("dense", 1, 0.5),
                                         ("tac", 4, 0.9), ("tactp", 4, 0.5)])
@pytest.mark.parametrize("case", LAYER_CASES, ids=[c[0] for c in LAYER_CASES])
def test_layer_parity(T, O, case, mode, K, beta, engine):
    name, (Tn, B, Cin, H, W, Cout, pad, pool), gain, rho = case
    spec = T.LayerSpec(T=Tn, B=B, C_in=Cin, H=H, W=W, C_out=Cout, pad=pad, K=K, mode=mode,
                       beta=beta, out_pool=pool)
    spec = _engine_or_skip(spec, engine)
    S = _spikes(zlib.crc32(name.encode()) % 1000, (Tn, B, Cin, H, W), rho)
    w, b = _w(7, Cout, Cin, gain)
    _, _, st = P.check_layer(T, O, spec, S, w, b, label=f"{name}/{mode}/K{K}/{engine}")
    assert 0.0 < st["rate"] < 0.9, st


SPLIT_CASES = [
    # beta != 2^-m (or m (K-1) > 7): A carried as fp16 hi + lo on the tensor cores
    ("C1", (8, 4, 1, 28, 28, 8, 0, 1), 2.5, 0.1),             # LDG producer, C_in 1
    ("mnistL1", (8, 3, 1, 28, 28, 32, 0, 2), 2.5, 0.15),
    ("mnistL2", (8, 3, 32, 13, 13, 64, 0, 1), 3.5, 0.15),     # LDG producer, C_in 32
    ("dvsL1s", (8, 2, 2, 64, 64, 128, 1, 2), 7.1, 0.05),       # TMA producer, C_in 2
    ("cin32_tma", (8, 2, 32, 12, 16, 64, 1, 2), 2.5, 0.15),   # TMA producer, C_in 32
]


@pytest.mark.parametrize("mode,K,beta", [("tac", 2, 0.9), ("tac", 4, 0.9), ("tac", 8, 0.9),
                                         ("tactp", 4, 0.9), ("tactp", 8, 0.25)])
@pytest.mark.parametrize("case", SPLIT_CASES, ids=[c[0] for c in SPLIT_CASES])
def test_split_aggregate_parity(T, O, case, mode, K, beta):
    """tcgen05 path with the split fp16 aggregate (the rate-coded configs' beta = 0.9)."""
    name, (Tn, B, Cin, H, W, Cout, pad, pool), gain, rho = case
    spec = T.LayerSpec(T=Tn, B=B, C_in=Cin, H=H, W=W, C_out=Cout, pad=pad, K=K, mode=mode,
                       beta=beta, out_pool=pool, engine="tcgen05")
    assert spec.engine_used() == "tcgen05"
    S = _spikes(zlib.crc32(name.encode()) % 997, (Tn, B, Cin, H, W), rho)
    w, b = _w(8, Cout, Cin, gain)
    _, _, st = P.check_layer(T, O, spec, S, w, b, label=f"split/{name}/{mode}/K{K}/b{beta}")
    assert 0.0 < st["rate"] < 0.9, st


REAL_CASES = [
    # continuous-valued first layer (log-normalised DVS-like event counts)
    ("dvsL1r", (8, 2, 2, 64, 64, 128, 1, 2), 4.0),
    ("mnistL1r", (8, 3, 1, 28, 28, 32, 0, 2), 2.5),
    ("c1r", (8, 4, 1, 28, 28, 8, 0, 1), 2.5),
]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("mode,K,beta", [("dense", 1, 0.5), ("tac", 4, 0.5), ("tactp", 2, 0.9),
                                         ("tac", 8, 0.9), ("tactp", 4, 0.5)])
@pytest.mark.parametrize("case", REAL_CASES, ids=[c[0] for c in REAL_CASES])
def test_real_input_parity(T, O, case, mode, K, beta, engine):
    """tac_conv_lif_forward_real against the fp64 oracle on the same float frames."""
    from paper_2603_13810_b200 import synth
    name, (Tn, B, Cin, H, W, Cout, pad, pool), gain = case
    spec = T.LayerSpec(T=Tn, B=B, C_in=Cin, H=H, W=W, C_out=Cout, pad=pad, K=K, mode=mode,
                       beta=beta, out_pool=pool, input="real")
    spec = _engine_or_skip(spec, engine)
    X = synth.dvs_log_counts(zlib.crc32(name.encode()) % 991, Tn, B, H, W)[:, :, :Cin]  # [T,B,C,H,W]
    w, b = _w(10, Cout, Cin, gain)
    prep = T.prepare_weights(spec, w, b)
    x = X.permute(0, 1, 3, 4, 2).contiguous().cuda()                                   # [T,B,H,W,C]
    s1 = spec.replace(out_pool=1)
    out, vf, cnt = T.conv_lif(s1, prep, x, want_v_final=True)
    torch.cuda.synchronize()
    hc, wc = s1.conv_hw
    D = O.unpack_spikes(P.to_u32(out), Cout, wc)
    r = O.forward(X.numpy().astype(np.float64), w.numpy(), b.numpy(), K=s1.K, mode=mode,
                  beta=beta, pad=pad, replay=D, band=P.BAND)
    assert r["mismatch"] == 0, f"{name}: {r['mismatch']} out-of-band mismatches"
    assert 0.0 < D.mean() < 0.9, D.mean()
    v_dev = vf.cpu().numpy().transpose(0, 3, 1, 2).astype(np.float64)
    err = np.abs(v_dev - r["v_final"])
    assert np.all(err <= P.VTOL * np.maximum(np.abs(r["v_final"]), 1.0)), err.max()
    assert np.array_equal(cnt.cpu().numpy().astype(np.int64), r["counts"])
    if pool == 2:
        dev_p, _, _ = T.conv_lif(spec, prep, x, want_counts=False)
        torch.cuda.synchronize()
        assert np.array_equal(O.unpack_spikes(P.to_u32(dev_p), Cout, wc // 2), O.or_pool2(r["out"]))


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("mode", ["tac", "tactp"])
def test_real_input_partial_last_group(T, O, mode, engine):
    """Continuous input with K not dividing T (T = 10, K = 4: groups 4, 4, 2)."""
    from paper_2603_13810_b200 import synth
    Tn, B, Cin, H, W, Cout = 10, 2, 2, 32, 32, 128
    spec = T.LayerSpec(T=Tn, B=B, C_in=Cin, H=H, W=W, C_out=Cout, pad=1, K=4, mode=mode, beta=0.5,
                       out_pool=1, input="real", partial=True)
    spec = _engine_or_skip(spec, engine)
    X = synth.dvs_log_counts(5, Tn, B, H, W)                                   # [T,B,C,H,W]
    w, b = _w(15, Cout, Cin, 4.0)
    prep = T.prepare_weights(spec, w, b)
    out, vf, cnt = T.conv_lif(spec, prep, X.permute(0, 1, 3, 4, 2).contiguous().cuda(),
                              want_v_final=True)
    torch.cuda.synchronize()
    D = O.unpack_spikes(P.to_u32(out), Cout, W)
    r = O.forward(X.numpy().astype(np.float64), w.numpy(), b.numpy(), K=4, mode=mode, beta=0.5,
                  pad=1, replay=D, band=P.BAND, partial=True)
    assert r["mismatch"] == 0 and 0.0 < D.mean() < 0.9
    err = np.abs(vf.cpu().numpy().transpose(0, 3, 1, 2) - r["v_final"])
    assert np.all(err <= P.VTOL * np.maximum(np.abs(r["v_final"]), 1.0))
    assert np.array_equal(cnt.cpu().numpy().astype(np.int64), r["counts"])


def test_real_input_rejects_spike_call(T):
    """A REAL-input descriptor through tac_conv_lif_forward is refused before launch."""
    import ctypes
    spec = T.LayerSpec(T=4, B=1, C_in=2, H=8, W=8, C_out=16, pad=1, K=2, mode="tac", beta=0.5,
                       input="real")
    prep = T.prepare_weights(spec, *_w(1, 16, 2, 1.0))
    x = T.pack(torch.zeros((4, 1, 2, 8, 8), dtype=torch.uint8, device="cuda"))
    d = spec.desc()
    out = torch.empty((2, 1, 4, 16), dtype=torch.int32, device="cuda")
    st = T.lib().tac_conv_lif_forward(ctypes.byref(d), ctypes.byref(prep.plan),
                                      ctypes.c_void_p(x.data_ptr()), None,
                                      ctypes.c_void_p(out.data_ptr()), None, None, None, 0, None)
    assert st == 4 and b"tac_conv_lif_forward_real" in T.lib().tac_last_error_detail()


PARTIAL_CASES = [
    # (T, K): last group of K' = T - (G-1) K frames (the paper's T = 25)
    ("T10K4", 10, 4), ("T6K4", 6, 4), ("T3K4", 3, 4), ("T25K8", 25, 8),
]
PARTIAL_LAYERS = [
    ("int8", (2, 32, 12, 16, 64, 1, 2), 0.5, 2.5),       # C_in 32, exact aggregate
    ("fp16", (2, 2, 32, 32, 128, 1, 2), 0.5, 6.0),       # first layer, packed slices
    ("split", (2, 1, 28, 28, 32, 0, 2), 0.9, 2.5),       # beta = 0.9 split aggregate
]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("mode", ["tac", "tactp"])
@pytest.mark.parametrize("layer", PARTIAL_LAYERS, ids=[c[0] for c in PARTIAL_LAYERS])
@pytest.mark.parametrize("tk", PARTIAL_CASES, ids=[c[0] for c in PARTIAL_CASES])
def test_partial_last_group_parity(T, O, tk, layer, mode, engine):
    """K need not divide T (desc.partial_last_group): against the oracle's short-group
    semantics, on the path each layer type takes."""
    _, Tn, K = tk
    name, (B, Cin, H, W, Cout, pad, pool), beta, gain = layer
    spec = T.LayerSpec(T=Tn, B=B, C_in=Cin, H=H, W=W, C_out=Cout, pad=pad, K=K, mode=mode,
                       beta=beta, out_pool=pool, partial=True)
    spec = _engine_or_skip(spec, engine)
    S = _spikes(zlib.crc32((name + tk[0]).encode()) % 977, (Tn, B, Cin, H, W), 0.15)
    w, b = _w(12, Cout, Cin, gain)
    _, _, st = P.check_layer(T, O, spec, S, w, b, label=f"partial/{tk[0]}/{name}/{mode}/{engine}")
    assert 0.0 < st["rate"] < 0.95, st


@pytest.mark.parametrize("mode", ["tac", "tactp"])
@pytest.mark.parametrize("layer", PARTIAL_LAYERS, ids=[c[0] for c in PARTIAL_LAYERS])
def test_group_size_3_on_tcgen05(T, O, layer, mode):
    """K = 3 (short last groups such as T = 7, K = 4) runs on the tcgen05 engine."""
    name, (B, Cin, H, W, Cout, pad, pool), beta, gain = layer
    spec = T.LayerSpec(T=6, B=B, C_in=Cin, H=H, W=W, C_out=Cout, pad=pad, K=3, mode=mode,
                       beta=beta, out_pool=pool, engine="tcgen05")
    assert spec.engine_used() == "tcgen05"
    S = _spikes(zlib.crc32(name.encode()) % 971, (6, B, Cin, H, W), 0.15)
    w, b = _w(13, Cout, Cin, gain)
    _, _, st = P.check_layer(T, O, spec, S, w, b, label=f"K3/{name}/{mode}")
    assert 0.0 < st["rate"] < 0.95, st


@pytest.mark.parametrize("mode", ["tac", "tactp"])
def test_odd_group_size_runs_on_simt(T, O, mode):
    """K = 5 (T = 10) is outside the tcgen05 envelope (K in {1,2,3,4,8}): AUTO must pick
    the SIMT engine, an explicit tcgen05 request must be refused, results exact."""
    spec = T.LayerSpec(T=10, B=2, C_in=32, H=10, W=12, C_out=32, pad=1, K=5, mode=mode,
                       beta=0.5, out_pool=2)
    assert spec.engine_used() == "simt"
    with pytest.raises(RuntimeError):
        spec.replace(engine="tcgen05").engine_used()
    S = _spikes(21, (10, 2, 32, 10, 12), 0.2)
    w, b = _w(9, 32, 32, 1.5)
    P.check_layer(T, O, spec, S, w, b, label=f"K5/{mode}")


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("reset", ["delayed", "hard"])
@pytest.mark.parametrize("mode", ["dense", "tac", "tactp"])
def test_reset_variants(T, O, mode, reset, engine):
    spec = T.LayerSpec(T=8, B=3, C_in=32, H=12, W=12, C_out=32, pad=1, K=2, mode=mode,
                       beta=0.5, v_reset=-0.25, reset=reset, out_pool=2)
    spec = _engine_or_skip(spec, engine)
    S = _spikes(11, (8, 3, 32, 12, 12), 0.2)
    w, b = _w(3, 32, 32, 1.5)
    P.check_layer(T, O, spec, S, w, b, label=f"{mode}/{reset}/{engine}")


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("reset", ["subtract", "delayed", "hard"])
@pytest.mark.parametrize("shape", ["int8", "fp16_first"])
def test_v_init_chaining(T, O, reset, engine, shape):
    """P12 on the device: forward(T) == forward(T1) -> forward(T-T1, v_init=v_final),
    bitwise on every path (int8 32->32, and the fp16 first-layer path 2->128 with TAC-TP
    K=4 whose subtract-reset state lives in TMEM)."""
    cin, cout, K, gain = (32, 32, 2, 1.2) if shape == "int8" else (2, 128, 4, 3.0)
    spec = T.LayerSpec(T=8, B=2, C_in=cin, H=10, W=10, C_out=cout, pad=1, K=K, mode="tactp",
                       beta=0.5, reset=reset, out_pool=1)
    spec = _engine_or_skip(spec, engine)
    S = _spikes(12, (8, 2, cin, 10, 10), 0.25)
    w, b = _w(4, cout, cin, gain)
    prep = T.prepare_weights(spec, w, b)
    x = T.pack(torch.from_numpy(S).cuda())
    full, vf, _ = T.conv_lif(spec, prep, x, want_v_final=True)
    h = spec.replace(T=4)
    a, va, _ = T.conv_lif(h, prep, x[:4], want_v_final=True)
    c, vc, _ = T.conv_lif(h, prep, x[4:], v_init=va, want_v_final=True)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat([a, c]), full)
    # every path carries V itself across the call boundary (the tcgen05 subtract-reset
    # epilogue keeps V scaled by the power of two 2^e, which is exact): bit-exact
    assert torch.equal(vc, vf)
    # and the chained second half against the oracle with v_init
    P.check_layer(T, O, h, S[4:], w, b, v_init=va.cpu().numpy().transpose(0, 3, 1, 2),
                  label=f"chain/{reset}/{engine}")


@pytest.mark.parametrize("engine", ENGINES)
def test_exhaustive_tiny_batch(T, O, engine):
    """P9: every binary input of a 1-channel 2x2 image over T=4 steps (2^16
    samples in one batch), pad 1, K=2, all three modes."""
    bits = np.array(list(itertools.product([0, 1], repeat=16)), np.uint8)   # [65536, 16]
    S = np.ascontiguousarray(bits.reshape(-1, 4, 1, 2, 2).transpose(1, 0, 2, 3, 4))
    w, b = _w(5, 16, 1, 3.0)
    for mode in ("dense", "tac", "tactp"):
        spec = T.LayerSpec(T=4, B=S.shape[1], C_in=1, H=2, W=2, C_out=16, pad=1, K=2,
                           mode=mode, beta=0.5, out_pool=1)
        spec = _engine_or_skip(spec, engine)
        P.check_layer(T, O, spec, S, w, b, label=f"exhaustive/{mode}/{engine}")


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("reset", ["subtract", "delayed", "hard"])
@pytest.mark.parametrize("mode", ["dense", "tac", "tactp"])
def test_exhaustive_batch_bitwise_vs_bruteforce(T, mode, reset, engine):
    """P9, device vs the independent brute force (tests/bruteforce.py) on all 2^16 inputs:
    weights n/64 with max |n| = 127 are exact in both tensor-core operand formats (int8
    slice step max|w|/127 = 1/64; fp16), beta = 1/2 and the small binary fractions keep every
    sum exact in fp32 -- so spikes, counts and v_final must agree BITWISE, no band."""
    import bruteforce
    bits = np.array(list(itertools.product([0, 1], repeat=16)), np.uint8)
    S = np.ascontiguousarray(bits.reshape(-1, 4, 1, 2, 2).transpose(1, 0, 2, 3, 4))
    rng = np.random.default_rng(11)
    n = rng.integers(-100, 101, (16, 1, 3, 3))
    n[:, 0, 1, 1] = 127                                        # max |n| = 127 in every channel
    w = torch.from_numpy((n / 64.0).astype(np.float32) * 0.5)  # 0.5 n/64 = n/128: still exact
    b = torch.from_numpy((rng.integers(-4, 5, 16) / 16.0).astype(np.float32))
    spec = T.LayerSpec(T=4, B=S.shape[1], C_in=1, H=2, W=2, C_out=16, pad=1, K=2, mode=mode,
                       beta=0.5, v_reset=-0.25, reset=reset, out_pool=1)
    spec = _engine_or_skip(spec, engine)
    prep = T.prepare_weights(spec, w, b)
    out, vf, cnt = T.conv_lif(spec, prep, T.pack(torch.from_numpy(S).cuda()), want_v_final=True)
    torch.cuda.synchronize()
    ref, V = bruteforce.layer(S, w.numpy(), b.numpy(), K=2, mode=mode, beta=0.5, v_th=1.0,
                              reset=reset, v_reset=-0.25, pad=1)
    from oracle import oracle as O
    D = O.unpack_spikes(P.to_u32(out), 16, 2)
    assert 0.02 < ref.mean() < 0.98
    assert np.array_equal(D, ref)
    assert np.array_equal(vf.cpu().numpy().transpose(0, 3, 1, 2).astype(np.float64), V)
    assert np.array_equal(cnt.cpu().numpy().astype(np.int64), ref.sum(axis=(0, 3, 4)))


def test_plan_mismatch_refused(T):
    """tac_plan: weights prepared for TAC and run as TAC-TP (different folded bias and
    aggregate scale) are refused with TAC_ERR_PARAM before any launch; a batch shard of the
    same layer (different B) is accepted."""
    spec = T.LayerSpec(T=8, B=4, C_in=32, H=12, W=12, C_out=32, pad=1, K=4, mode="tac", beta=0.5)
    prep = T.prepare_weights(spec, *_w(2, 32, 32, 1.0))
    x = T.pack(torch.zeros((8, 4, 32, 12, 12), dtype=torch.uint8, device="cuda"))
    for bad in (spec.replace(mode="tactp"), spec.replace(K=2), spec.replace(beta=0.25),
                spec.replace(v_th=2.0), spec.replace(reset="hard"), spec.replace(pad=0),
                spec.replace(agg_weights=(0.125, 0.25, 0.5, 1.0))):
        with pytest.raises(RuntimeError, match="TAC_ERR_PARAM.*different descriptor"):
            T.conv_lif(bad, prep, x if bad.pad == 1 else x)
    T.conv_lif(spec.replace(B=2), prep, x[:, :2])       # batch shard: same image
    T.conv_lif(spec.replace(T=4), prep, x[:4])           # chunked sequence: same image
    torch.cuda.synchronize()


ALPHA_CASES = [
    # learnable aggregation weights alpha_j: split (table) path on tcgen05
    ("c1", (8, 3, 1, 28, 28, 32, 0, 2), 2.5),
    ("c2", (8, 2, 2, 32, 32, 128, 1, 2), 6.0),
    ("c32", (8, 2, 32, 12, 16, 64, 1, 2), 2.5),
    ("c128_simt", (8, 2, 128, 8, 8, 128, 1, 2), 3.0),   # outside the split envelope: SIMT
]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("mode,K,alpha", [("tac", 4, (0.3, -0.2, 1.1, 0.7)),
                                          ("tactp", 2, (0.45, 0.9)),
                                          ("tac", 8, (0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8))])
@pytest.mark.parametrize("case", ALPHA_CASES, ids=[c[0] for c in ALPHA_CASES])
def test_agg_weights_parity(T, O, case, mode, K, alpha, engine):
    name, (Tn, B, Cin, H, W, Cout, pad, pool), gain = case
    spec = T.LayerSpec(T=Tn, B=B, C_in=Cin, H=H, W=W, C_out=Cout, pad=pad, K=K, mode=mode,
                       beta=0.9, out_pool=pool, agg_weights=alpha)
    if name.endswith("simt") and engine == "tcgen05":
        with pytest.raises(RuntimeError):
            spec.replace(engine="tcgen05").engine_used()
        return
    spec = _engine_or_skip(spec, engine)
    S = _spikes(zlib.crc32(name.encode()) % 983, (Tn, B, Cin, H, W), 0.15)
    w, b = _w(16, Cout, Cin, gain)
    _, _, st = P.check_layer(T, O, spec, S, w, b, label=f"alpha/{name}/{mode}/K{K}/{engine}")
    assert 0.0 < st["rate"] < 0.95, st


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("mode", ["tac", "tactp"])
def test_agg_weights_partial_last_group(T, O, mode, engine):
    """T = 10, K = 4 with alpha: the short group (2 frames) uses alpha_2, alpha_3 (reading R11)."""
    spec = T.LayerSpec(T=10, B=2, C_in=2, H=24, W=24, C_out=64, pad=1, K=4, mode=mode, beta=0.9,
                       out_pool=2, partial=True, agg_weights=(0.2, 0.4, -0.3, 0.9))
    spec = _engine_or_skip(spec, engine)
    S = _spikes(77, (10, 2, 2, 24, 24), 0.2)
    w, b = _w(17, 64, 2, 5.0)
    _, _, st = P.check_layer(T, O, spec, S, w, b, label=f"alpha-partial/{mode}/{engine}")
    assert 0.0 < st["rate"] < 0.95, st


RUNTIME_K = [5, 6, 7, 9, 12, 16]


@pytest.mark.parametrize("beta", [0.9, 0.5])
@pytest.mark.parametrize("K", RUNTIME_K)
@pytest.mark.parametrize("cin", [1, 2])
def test_runtime_group_size_on_tcgen05(T, O, cin, K, beta):
    """Any K <= 16 on the first layers (split table path, runtime-K producers; K > 8 uses the
    two fp32 half tables): TAC (and TAC-TP for K <= 8) against the oracle."""
    Tn = 2 * K
    H, W, Cout = (28, 28, 32) if cin == 1 else (32, 32, 128)
    for mode in (["tac", "tactp"] if K <= 8 else ["tac"]):
        spec = T.LayerSpec(T=Tn, B=2, C_in=cin, H=H, W=W, C_out=Cout, pad=0 if cin == 1 else 1,
                           K=K, mode=mode, beta=beta, out_pool=2, engine="tcgen05")
        assert spec.engine_used() == "tcgen05"
        S = _spikes(K * 10 + cin, (Tn, 2, cin, H, W), 0.12)
        w, b = _w(18, Cout, cin, 2.0 if mode == "tac" else 1.0)
        _, _, st = P.check_layer(T, O, spec, S, w, b, label=f"K{K}/{cin}/{mode}/b{beta}")
        assert 0.0 < st["rate"] < 0.95, st


@pytest.mark.parametrize("K", [16, 8, 4])
def test_mnist_T25_on_tcgen05(T, O, K):
    """The paper's MNIST setting T = 25 with K = 4/8/16: partial last
    groups (K' = 1, 1, 9), every layer of the C2-shaped stack on the tensor cores."""
    from paper_2603_13810_b200 import configs
    cfg = configs.CONFIGS["C2"]
    specs = configs.layer_plan(cfg, mode="tac", K=K, B=3, T=25, engine="tcgen05")
    assert all(s.engine_used() == "tcgen05" for s in specs), [s.engine_used() for s in specs]
    S = configs.make_inputs(cfg, B=3, T=25).numpy()
    stats = P.check_stack(T, O, specs, configs.layer_weights(cfg), S, label=f"C2@T25/K{K}")
    assert stats[0]["rate"] > 0.0


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("scale", [1e-4, 1.0, 300.0])
def test_fp16_operand_prescale(T, O, scale, engine):
    """The fp16 operand paths prescale the layer by 2^e (tc_prepare): weights, bias and v_th
    scaled together by `scale` (far from 1 both ways) give the same spikes as scale 1, and
    parity with the oracle holds (no absolute 2^-24 quantum, no fp16 overflow)."""
    for cin, beta, K in ((2, 0.5, 4), (1, 0.9, 4)):
        spec = T.LayerSpec(T=8, B=2, C_in=cin, H=20, W=20, C_out=32, pad=1, K=K, mode="tactp",
                           beta=beta, v_th=scale, v_reset=0.0, out_pool=1)
        spec = _engine_or_skip(spec, engine)
        w, b = _w(19, 32, cin, 4.0)
        S = _spikes(5 + cin, (8, 2, cin, 20, 20), 0.2)
        _, _, st = P.check_layer(T, O, spec, S, w * scale, b * scale,
                                 label=f"prescale/{scale}/{cin}/{engine}")
        assert 0.0 < st["rate"] < 0.95, st


def test_shard_invariance(T):
    """P13: a batch-shard view gives bitwise the same per-sample outputs."""
    spec = T.LayerSpec(T=8, B=6, C_in=128, H=16, W=16, C_out=128, pad=1, K=4, mode="tactp",
                       beta=0.5, out_pool=2)
    S = _spikes(13, (8, 6, 128, 16, 16), 0.1)
    w, b = _w(6, 128, 128, 1.0)
    prep = T.prepare_weights(spec, w, b)
    x = T.pack(torch.from_numpy(S).cuda())
    full, vf, cf = T.conv_lif(spec, prep, x, want_v_final=True)
    parts = [T.conv_lif(spec.replace(B=3), prep, x[:, i:i + 3], want_v_final=True)
             for i in (0, 3)]
    torch.cuda.synchronize()
    assert torch.equal(torch.cat([p[0] for p in parts], 1), full)
    assert torch.equal(torch.cat([p[1] for p in parts], 0), vf)
    assert torch.equal(torch.cat([p[2] for p in parts], 0), cf)


def test_errors_launch_nothing(T):
    spec = T.LayerSpec(T=8, B=2, C_in=2, H=8, W=8, C_out=16, pad=1, K=4, mode="tac", beta=0.5)
    prep = T.prepare_weights(spec, *_w(1, 16, 2, 1.0))
    x = T.pack(torch.zeros((8, 2, 2, 8, 8), dtype=torch.uint8, device="cuda"))
    with pytest.raises(RuntimeError, match="K_NOT_DIVIDING"):
        T.conv_lif(spec.replace(K=3), prep, x)
    with pytest.raises(RuntimeError, match="NONFINITE"):
        w, b = _w(1, 16, 2, 1.0)
        w[0, 0, 0, 0] = float("nan")
        T.prepare_weights(spec, w, b)
    xc = x.cpu()
    import ctypes
    d = spec.desc()
    out = torch.empty((2, 2, 8, 4), dtype=torch.int32, device="cuda")
    st = T.lib().tac_conv_lif_forward(ctypes.byref(d), ctypes.byref(prep.plan),
                                      ctypes.c_void_p(xc.data_ptr()), None,
                                      ctypes.c_void_p(out.data_ptr()), None, None, None, 0, None)
    assert st == 4 and b"not device memory" in T.lib().tac_last_error_detail()


# ------------------------------------------------------------- stacks -------
@pytest.mark.parametrize("cfg_name,B,mode", [("C1", 4, "tac"), ("C1", 4, "dense"),
                                             ("C2", 6, "tac"), ("C3", 4, "tac"),
                                             ("C3", 2, "dense"), ("C4", 2, "tactp"),
                                             ("C4", 1, "tac"), ("C4", 1, "dense")])
def test_config_stack_parity(T, O, cfg_name, B, mode):
    from paper_2603_13810_b200 import configs
    cfg = configs.CONFIGS[cfg_name]
    specs = configs.layer_plan(cfg, mode=mode, B=B)
    if mode == "tac" and cfg.inputs == "dvs":
        specs = configs.layer_plan(cfg, mode=mode, K=2, B=B)[:4]   # 16/2^4 = 1 step left
    weights = configs.layer_weights(cfg, mode=mode)[:len(specs)]   # mode-specific gains
    S = configs.make_inputs(cfg, B=B).numpy()
    stats = P.check_stack(T, O, specs, weights, S, label=f"{cfg_name}/{mode}")
    # every layer fires (the DVS dense stack runs with its own calibrated gains, so its
    # deep-layer parity is not vacuous); the last layer of a short C1 / MNIST run may be sparse
    for i, st in enumerate(stats):
        assert st["rate"] > (0.005 if cfg.inputs == "dvs" else 0.0), (i, st["rate"])


@pytest.mark.parametrize("reset", ["subtract", "delayed", "hard"])
@pytest.mark.parametrize("mode,K", [("dense", 1), ("tac", 4), ("tactp", 2)])
def test_fc_layer_parity(T, O, mode, K, reset):
    """Fully connected LIF layer (1x1 conv of a 1x1 image; SIMT fc kernel), C_in not a
    multiple of 32 and C_out spanning two spike words."""
    spec = T.LayerSpec(T=8, B=5, C_in=200, H=1, W=1, C_out=40, R=1, S=1, pad=0, K=K, mode=mode,
                       beta=0.9, v_reset=-0.2, reset=reset)
    S = _spikes(31, (8, 5, 200, 1, 1), 0.2)
    w, b = _w(14, 40, 200, 3.0, r=1, s=1)
    _, _, st = P.check_layer(T, O, spec, S, w, b, label=f"fc/{mode}/{reset}")
    assert 0.0 < st["rate"] < 0.95, st


# FC shapes of both whole networks on the tcgen05 FC kernel (fc.cu) and the SIMT one:
# C_in, C_out, B (ragged 128-sample M tiles), T, mode, K, beta
FC_CASES = [(1600, 128, 130, 8, "tac", 4, 0.9), (2048, 512, 40, 8, "tactp", 4, 0.5),
            (512, 110, 3, 6, "dense", 1, 0.5), (128, 10, 5, 4, "tac", 2, 0.9),
            (96, 40, 7, 6, "tactp", 2, 0.9), (200, 64, 257, 8, "tactp", 8, 0.5)]


@pytest.mark.parametrize("engine", ["simt", "tcgen05", "tcgen05-fused"])
@pytest.mark.parametrize("reset", ["subtract", "delayed", "hard"])
@pytest.mark.parametrize("case", FC_CASES, ids=lambda c: f"{c[0]}x{c[1]}b{c[2]}{c[4]}{c[5]}")
def test_fc_engines_parity(T, O, case, reset, engine):
    """Fully connected LIF layers on both engines: the tcgen05 FC
    GEMM (M = 128 samples, fp16 hi + lo operands, aggregate table) -- two-phase (group
    GEMMs split over the SMs into the workspace, then the LIF) and, without a workspace,
    fused -- and the SIMT kernel."""
    c_in, c_out, B, Tn, mode, K, beta = case
    fused = engine == "tcgen05-fused"
    engine = "tcgen05" if fused else engine
    spec = T.LayerSpec(T=Tn, B=B, C_in=c_in, H=1, W=1, C_out=c_out, R=1, S=1, pad=0, K=K,
                       mode=mode, beta=beta, v_reset=-0.2, reset=reset)
    spec = _engine_or_skip(spec, engine)
    seed = zlib.crc32(repr(case).encode()) & 0xFFFF
    S = _spikes(seed, (Tn, B, c_in, 1, 1), 0.2)
    w, b = _w(seed + 1, c_out, c_in, 3.0, r=1, s=1)
    _, _, st = P.check_layer(T, O, spec, S, w, b, label=f"fc/{case}/{reset}/{engine}", workspace=not fused)
    assert 0.0 < st["rate"] < 0.95, st


def test_fc_tcgen05_envelope(T):
    """The FC shapes the whole networks use all run on tcgen05 (no silent SIMT fallback)."""
    from paper_2603_13810_b200 import configs
    for name in ("C2", "C3", "C4", "C5"):
        for mode in ("dense", "tac", "tactp"):
            for s in configs.network_plan(configs.CONFIGS[name], mode=mode, B=8):
                if s.H == 1:
                    assert s.engine_used() == "tcgen05", (name, mode, s)


@pytest.mark.parametrize("mode,K", [("tactp", 2), ("dense", 1)])
def test_whole_dvs_network_parity(T, O, mode, K):
    """SURVEY.md 8(f) #2, DVS: 5 conv blocks + FC(2048->512) + FC(512->110), layer by layer
    against the oracle, then the VotingLayer (10 voters, 11 classes) on the device counts
    against oracle.vote of the oracle counts."""
    from paper_2603_13810_b200 import configs
    cfg = configs.CONFIGS["C4"]
    specs = configs.network_plan(cfg, mode=mode, K=K, B=1)
    S = configs.make_inputs(cfg, B=1).numpy()
    stats = P.check_stack(T, O, specs, configs.network_weights(cfg, mode=mode), S, label=f"C4/net/{mode}")
    for i, st in enumerate(stats):
        assert st["rate"] > 0.005, (i, st["rate"])
    last = specs[-1]
    T_out = last.T if last.mode != "tac" else -(-last.T // last.K)
    counts = torch.from_numpy(stats[-1]["counts"].astype(np.int32)).cuda()
    scores = T.vote(counts, 10, T_out).cpu().numpy()
    ref = O.vote(stats[-1]["counts"], 10, T_out)
    assert scores.shape == (1, 11)
    np.testing.assert_allclose(scores, ref, rtol=1e-6, atol=0)


def test_vote_parity(T, O):
    """tac_vote against oracle.vote on random counts (exact u32 sums, one fp32 division)."""
    g = torch.Generator().manual_seed(5)
    counts = torch.randint(0, 33, (37, 110), generator=g, dtype=torch.int32)
    scores = T.vote(counts.cuda(), 10, 32).cpu().numpy()
    np.testing.assert_allclose(scores, O.vote(counts.numpy(), 10, 32), rtol=1e-6, atol=0)


@pytest.mark.parametrize("cfg_name,B,mode,K", [("C2", 6, "tac", 4), ("C2", 4, "dense", 1),
                                               ("C3", 4, "tac", 8), ("C2", 4, "tactp", 2)])
def test_whole_mnist_network_parity(T, O, cfg_name, B, mode, K):
    """conv stack + floor-pooled 5x5 map + FC(1600->128) + FC(128->10),
    layer by layer against the oracle (the FC layers run as 1x1 convs of a 1x1 image)."""
    from paper_2603_13810_b200 import configs
    cfg = configs.CONFIGS[cfg_name]
    specs = configs.network_plan(cfg, mode=mode, K=K, B=B)
    S = configs.make_inputs(cfg, B=B).numpy()
    stats = P.check_stack(T, O, specs, configs.network_weights(cfg), S, label=f"{cfg_name}/net/{mode}")
    assert stats[-1]["rate"] > 0.0


def test_graph_replay_equals_eager(T):
    """Network.capture: a CUDA-graph replay of the stack gives bitwise the eager outputs
    (and refreshes them when the static input changes)."""
    from paper_2603_13810_b200 import configs, network
    cfg = configs.CONFIGS["C2"]
    net = network.Network(configs.network_plan(cfg, mode="tac", K=4, B=8), configs.network_weights(cfg))
    x = T.pack(configs.make_inputs(cfg, B=8, device="cuda"))
    y_eager, c_eager, _, _ = net.forward(x)
    graph, (y_g, c_g, _, _) = net.capture(x)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(y_g, y_eager) and torch.equal(c_g[-1], c_eager[-1])
    x.copy_(T.pack(configs.make_inputs(cfg, B=8, seed=1, device="cuda")))
    y2, c2, _, _ = net.forward(x)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(y_g, y2) and torch.equal(c_g[-1], c2[-1])
    assert not torch.equal(y2, y_eager) or not torch.equal(c2[-1], c_eager[-1])


@pytest.mark.slow
def test_c5_full_size_sampled(T, O):
    """C5 at its full batch (2048) in the bench launch configuration; sampled
    samples are re-checked layer by layer through the oracle replay, and the
    full-batch pooled outputs for those samples must equal the oracle's."""
    from paper_2603_13810_b200 import configs, network
    cfg = configs.CONFIGS["C5"]
    specs = configs.layer_plan(cfg)
    weights = configs.layer_weights(cfg)
    net = network.Network(specs, weights)
    x = T.pack(configs.make_inputs(cfg, device="cuda"))
    _, counts, outs, _ = net.forward(x, keep=True, want_counts=True)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    samples = [0, cfg.B - 1] + sorted(rng.choice(np.arange(1, cfg.B - 1), 2, replace=False).tolist())
    for bsel in samples:
        S = configs.make_inputs(cfg, B=1, b0=bsel).numpy()
        x_dev = None
        for i, (spec, (w, b)) in enumerate(zip(specs, weights)):
            s1 = spec.replace(B=1)
            ref_out, dev_out, st = P.check_layer(T, O, s1, S, w, b, x_packed=x_dev,
                                                 label=f"C5 sample {bsel} layer {i}")
            full_b = P.to_u32(outs[i][:, bsel:bsel + 1])
            assert np.array_equal(full_b, O.pack_spikes(ref_out)), f"layer {i} sample {bsel}"
            assert np.array_equal(counts[i][bsel].cpu().numpy().astype(np.int64),
                                  st["counts"][0]), f"counts layer {i} sample {bsel}"
            S, x_dev = ref_out, dev_out

