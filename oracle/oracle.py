"""CPU oracle for the Conv-LIF layer of arXiv 2603.13810 (TAC / TAC-TP / dense).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product package ``paper_2603_13810_b200`` never imports it, and the
two share no code: the arithmetic lives in ``oracle/tac_oracle.c`` (fp64, direct
loops, see its header for the paper citations); this file is ctypes marshalling
plus plain numpy reference implementations of the packed spike format (row a0 of
SURVEY.md section 8, defined in include/tacsnn.h) and the OR-pool.

Citations "P:n" are /root/reference/PAPER.md line n, "S:n" SPEC.md line n.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tac_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

MODES = {"dense": 0, "tac": 1, "tactp": 2}
RESETS = {"subtract": 0, "delayed": 1, "hard": 2}


def build(force: bool = False) -> str:
    """Compile oracle/tac_oracle.c into oracle/liboracle.so (gcc, OpenMP)."""
    if force or not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC)):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared",
                               "-std=c11", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = ctypes.CDLL(build())
            P = ctypes.c_void_p
            i, d = ctypes.c_int, ctypes.c_double
            L.tac_oracle_forward.argtypes = [P, P, P] + [i] * 12 + [d, d, d, i] + \
                [P, P, P, P, P, d, P, P]
            L.tac_oracle_forward.restype = i
            L.tac_oracle_forward_x.argtypes = L.tac_oracle_forward.argtypes
            L.tac_oracle_forward_x.restype = i
            L.tac_oracle_forward_alpha.argtypes = [P, P, P] + L.tac_oracle_forward.argtypes[1:]
            L.tac_oracle_forward_alpha.restype = i
            L.tac_oracle_conv2d.argtypes = [P, P, P] + [i] * 9 + [P]
            L.tac_oracle_conv2d.restype = i
            L.tac_oracle_or_pool2.argtypes = [P, i, i, i, i, P]
            L.tac_oracle_or_pool2.restype = i
            L.tac_oracle_threads.restype = i
            L.tac_oracle_backward.argtypes = [P, P, P, P, P] + [i] * 12 + [d, d, i, d, i] + \
                [P, P, d, P, P, P, P, P, P, P]
            L.tac_oracle_backward.restype = i
            L.tac_oracle_set_threads.argtypes = [i]
            L.tac_oracle_set_threads.restype = None
            _lib = L
    return _lib


def threads() -> int:
    return int(lib().tac_oracle_threads())


def set_threads(n: int) -> None:
    """OpenMP threads of later oracle calls (single-core baseline timing)."""
    lib().tac_oracle_set_threads(int(n))


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def out_hw(H, W, R=3, S=3, stride=1, pad=0):
    return (H + 2 * pad - R) // stride + 1, (W + 2 * pad - S) // stride + 1


def conv2d(X, Wt, bias=None, stride=1, pad=0):
    """fp64 direct-loop cross-correlation.  X [B,Cin,H,W] -> [B,Cout,Ho,Wo]."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    Wt = np.ascontiguousarray(Wt, dtype=np.float32)
    bias = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    B, Cin, H, W = X.shape
    Cout, _, R, S = Wt.shape
    Ho, Wo = out_hw(H, W, R, S, stride, pad)
    Y = np.empty((B, Cout, Ho, Wo), np.float64)
    rc = lib().tac_oracle_conv2d(_ptr(X), _ptr(Wt), _ptr(bias), B, Cin, H, W, Cout,
                                 R, S, stride, pad, _ptr(Y))
    assert rc == 0
    return Y


def forward(S, Wt, bias=None, *, K=1, mode="tac", beta=0.9, v_th=1.0, v_reset=0.0,
            reset="subtract", stride=1, pad=0, v_init=None, replay=None, band=1e-3,
            partial=False, alpha=None):
    """One Conv-LIF layer (Eq. 1 / Alg. 1 / Alg. 2) on u8 spikes S [T,B,Cin,H,W]
    or, when S is a floating array, on continuous-valued input frames (computed
    in fp64; the DVS first layer's log-normalised counts).

    Returns dict(out u8 [T_out,B,Cout,Ho,Wo], v_final f64 [B,Cout,Ho,Wo],
    counts i64 [B,Cout], mismatch, excused).  ``beta``/``v_th``/``v_reset`` are
    rounded to fp32 first (the layer's parameters are fp32 in the ABI) and then
    used in fp64.  With ``replay`` (device spikes, same layout as out) the
    trajectory follows the replay protocol described in tac_oracle.c.
    ``alpha`` (K values, rounded to fp32 like the ABI's agg_weights): learnable
    aggregation weights in place of beta^{K-1-j} (reading R11).
    """
    real = np.issubdtype(np.asarray(S).dtype, np.floating)
    S = np.ascontiguousarray(S, dtype=np.float64 if real else np.uint8)
    Wt = np.ascontiguousarray(Wt, dtype=np.float32)
    bias = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    T, B, Cin, H, W = S.shape
    Cout, Cin2, R, Sk = Wt.shape
    assert Cin2 == Cin
    m = MODES[mode]
    if m == 0:
        K = 1
    if T % K and not partial:
        raise ValueError(f"K={K} does not divide T={T}")
    Ho, Wo = out_hw(H, W, R, Sk, stride, pad)
    T_out = -(-T // K) if m == 1 else T   # partial=True: ceil(T/K) groups, the last one short
    out = np.empty((T_out, B, Cout, Ho, Wo), np.uint8)
    v_final = np.empty((B, Cout, Ho, Wo), np.float64)
    counts = np.empty((B, Cout), np.int64)
    if v_init is not None:
        v_init = np.ascontiguousarray(v_init, dtype=np.float64)
        assert v_init.shape == (B, Cout, Ho, Wo)
    if replay is not None:
        replay = np.ascontiguousarray(replay, dtype=np.uint8)
        assert replay.shape == out.shape, (replay.shape, out.shape)
    mism = np.zeros(1, np.int64)
    exc = np.zeros(1, np.int64)
    f32 = lambda v: float(np.float32(v))
    L = lib()
    if alpha is not None:
        alpha = np.ascontiguousarray(np.asarray(alpha, np.float32).astype(np.float64))
        assert alpha.shape == (K,), (alpha.shape, K)
        fwd = lambda S_, *rest: L.tac_oracle_forward_alpha(
            None if real else S_, S_ if real else None, _ptr(alpha), *rest)
    else:
        fwd = L.tac_oracle_forward_x if real else L.tac_oracle_forward
    rc = fwd(
        _ptr(S), _ptr(Wt), _ptr(bias), T, B, Cin, H, W, Cout, R, Sk, stride, pad,
        -K if (partial and m != 0) else K, m,
        f32(beta), f32(v_th), f32(v_reset), RESETS[reset], _ptr(v_init), _ptr(out),
        _ptr(v_final), _ptr(counts), _ptr(replay), float(band), _ptr(mism), _ptr(exc))
    if rc != 0:
        raise ValueError("tac_oracle_forward rejected its arguments")
    return dict(out=out, v_final=v_final, counts=counts, mismatch=int(mism[0]),
                excused=int(exc[0]))


SURROGATES = {"fast_sigmoid": 0, "arctan": 1}


def backward(S, Wt, bias, g_out, *, K=1, mode="tac", beta=0.9, v_th=1.0, stride=1, pad=0,
             surrogate="fast_sigmoid", sg_alpha=25.0, detach_reset=False, v_init=None,
             g_vfinal=None, replay=None, band=1e-3, alpha=None, want_input=True):
    """Surrogate-gradient BPTT of one Conv-LIF layer (subtract reset; see the
    backward section of tac_oracle.c for the equations and citations).
    S: u8 spikes or float frames [T,B,Cin,H,W]; g_out fp64 [T_out,B,Cout,Ho,Wo] = dL/ds.
    Returns dict(g_W [Cout,Cin,R,S], g_b [Cout], g_in [T,B,Cin,H,W] or None,
    g_vinit [B,Cout,Ho,Wo], g_alpha [K] or None), all fp64."""
    real = np.issubdtype(np.asarray(S).dtype, np.floating)
    S = np.ascontiguousarray(S, dtype=np.float64 if real else np.uint8)
    Wt = np.ascontiguousarray(Wt, dtype=np.float32)
    bias = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    T, B, Cin, H, W = S.shape
    Cout, _, R, Sk = Wt.shape
    m = MODES[mode]
    if m == 0:
        K = 1
    Ho, Wo = out_hw(H, W, R, Sk, stride, pad)
    g_out = np.ascontiguousarray(g_out, dtype=np.float64)
    g_W = np.empty((Cout, Cin, R, Sk))
    g_b = np.empty(Cout)
    g_in = np.empty((T, B, Cin, H, W)) if want_input else None
    g_vinit = np.empty((B, Cout, Ho, Wo))
    g_alpha = np.empty(K) if alpha is not None else None
    if alpha is not None:
        alpha = np.ascontiguousarray(np.asarray(alpha, np.float32).astype(np.float64))
    if v_init is not None:
        v_init = np.ascontiguousarray(v_init, dtype=np.float64)
    if g_vfinal is not None:
        g_vfinal = np.ascontiguousarray(g_vfinal, dtype=np.float64)
    if replay is not None:
        replay = np.ascontiguousarray(replay, dtype=np.uint8)
    f32 = lambda v: float(np.float32(v))
    rc = lib().tac_oracle_backward(
        None if real else _ptr(S), _ptr(S) if real else None, _ptr(alpha), _ptr(Wt), _ptr(bias),
        T, B, Cin, H, W, Cout, R, Sk, stride, pad, K, m, f32(beta), f32(v_th),
        SURROGATES[surrogate], float(sg_alpha), int(bool(detach_reset)), _ptr(v_init), _ptr(replay),
        float(band), _ptr(g_out), _ptr(g_vfinal), _ptr(g_W), _ptr(g_b), _ptr(g_in), _ptr(g_vinit),
        _ptr(g_alpha))
    if rc != 0:
        raise ValueError("tac_oracle_backward rejected its arguments")
    return dict(g_W=g_W, g_b=g_b, g_in=g_in, g_vinit=g_vinit, g_alpha=g_alpha)


def vote(counts, voters, T_out):
    """VotingLayer of the DVS network ("VotingLayer(10 voters, 11 classes)",
    :595): class j's score is the mean firing rate of its voters j*voters .. j*voters +
    voters - 1, i.e. their spike counts summed and divided by voters * T_out (fp64)."""
    counts = np.asarray(counts, dtype=np.float64)
    B, C = counts.shape
    assert C % voters == 0
    return counts.reshape(B, C // voters, voters).sum(axis=2) / (voters * T_out)


def or_pool2(x):
    """2x2 OR-pool of binary maps (P:235 MaxPool(2) on {0,1}); x [..., C, H, W].
    Odd extents: floor mode (the last row / column is dropped, as MaxPool2d)."""
    x = np.asarray(x, dtype=np.uint8)
    x = np.ascontiguousarray(x[..., : x.shape[-2] // 2 * 2, : x.shape[-1] // 2 * 2])
    *lead, C, H, W = x.shape
    N = int(np.prod(lead)) if lead else 1
    y = np.empty((*lead, C, H // 2, W // 2), np.uint8)
    rc = lib().tac_oracle_or_pool2(_ptr(x), N, C, H, W, _ptr(y))
    if rc != 0:
        raise ValueError("odd extent for 2x2 pool")
    return y


# ---------------------------------------------------------------------------
# Packed spike format (include/tacsnn.h, "Packed spike layout"), numpy reference.
# u32 [T][B][H][WPR], WPR = ceil(W*C/32); bit (t,b,c,y,x) lives at row offset
# r = x*C + c: word r>>5, bit r&31 (LSB first); pad bits are zero.
# ---------------------------------------------------------------------------
def words_per_row(W, C):
    return (W * C + 31) // 32


def pack_spikes(dense):
    """u8 {0,1} [T,B,C,H,W] -> u32 [T,B,H,WPR]."""
    dense = np.asarray(dense, dtype=np.uint8)
    T, B, C, H, W = dense.shape
    wpr = words_per_row(W, C)
    rows = dense.transpose(0, 1, 3, 4, 2).reshape(T, B, H, W * C)
    padded = np.zeros((T, B, H, wpr * 32), np.uint8)
    padded[..., :W * C] = rows
    by = np.packbits(padded, axis=-1, bitorder="little")
    return np.ascontiguousarray(by).view("<u4").reshape(T, B, H, wpr)


def unpack_spikes(packed, C, W):
    """u32 [T,B,H,WPR] -> u8 [T,B,C,H,W] (inverse of pack_spikes)."""
    packed = np.ascontiguousarray(packed, dtype="<u4")
    T, B, H, wpr = packed.shape
    bits = np.unpackbits(packed.view(np.uint8).reshape(T, B, H, wpr * 4), axis=-1,
                         bitorder="little")[..., :W * C]
    return np.ascontiguousarray(bits.reshape(T, B, H, W, C).transpose(0, 1, 4, 2, 3))


def group_count(T, K, mode):
    """Conv calls of one layer: G = T/K (Alg. 1/2), T for dense (Eq. 1)."""
    return T if mode == "dense" else T // K


def temporal_extents(T, Ks, modes):
    """Per-layer input extents and total conv calls of a stacked net (App. B,
    P:470-483): TAC divides the running extent by K_l, TAC-TP / dense keep it."""
    ext, calls, t = [], 0, T
    for K, mode in zip(Ks, modes):
        if mode != "dense" and t % K:
            raise ValueError(f"extent {t} not divisible by K={K}")
        ext.append(t)
        calls += group_count(t, K, mode)
        if mode == "tac":
            t //= K
    return ext, calls, t
