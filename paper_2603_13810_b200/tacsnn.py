"""Python binding of libtacsnn (include/tacsnn.h) -- argument marshalling only.

Every step of the Conv-LIF path runs in the library's CUDA kernels; this module
turns torch tensors into device pointers / strides and the current CUDA stream
into the ``stream`` argument.  There is no fallback: if ``libtacsnn.so`` is
missing or a call returns a non-OK status, a RuntimeError is raised.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import threading

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libtacsnn.so")
# A/B experiments: TACSNN_LIB=<path> loads a variant build (build.py TACSNN_LIB_NAME)
LIB_PATH = os.environ.get("TACSNN_LIB", LIB_PATH)

MODES = {"dense": 0, "tac": 1, "tactp": 2}
RESETS = {"subtract": 0, "delayed": 1, "hard": 2}
ENGINES = {"auto": 0, "simt": 1, "tcgen05": 2}
ENGINE_NAMES = {v: k for k, v in ENGINES.items()}
INPUTS = {"spikes": 0, "real": 1}
ABI_VERSION = 3

EXPORTS = ("tac_desc_check", "tac_out_shape", "tac_select_engine", "tac_weights_bytes",
           "tac_prepare_weights", "tac_workspace_bytes", "tac_conv_lif_forward",
           "tac_conv_lif_forward_real",
           "tac_pack_spikes", "tac_unpack_spikes", "tac_status_string",
           "tac_last_error_detail", "tac_abi_version", "tac_last_launch_count",
           "tac_debug_set_trace", "tac_conv_lif_forward_train", "tac_backward_workspace_bytes",
           "tac_conv_lif_backward", "tac_or_pool2", "tac_or_pool2_backward", "tac_vote")
SURROGATES = {"fast_sigmoid": 0, "arctan": 1}


class Desc(ctypes.Structure):
    """Mirror of tac_conv_lif_desc."""
    _fields_ = [(n, ctypes.c_int32) for n in ("T", "B", "C_in", "H", "W", "C_out", "R", "S",
                                               "stride", "pad", "K", "mode")] + \
               [("beta", ctypes.c_float), ("v_th", ctypes.c_float), ("v_reset", ctypes.c_float),
                ("reset", ctypes.c_int32), ("out_pool", ctypes.c_int32), ("engine", ctypes.c_int32),
                ("in_stride_t", ctypes.c_int64), ("in_stride_b", ctypes.c_int64),
                ("out_stride_t", ctypes.c_int64), ("out_stride_b", ctypes.c_int64),
                ("input_kind", ctypes.c_int32), ("partial_last_group", ctypes.c_int32),
                ("agg_weights", ctypes.POINTER(ctypes.c_float))]


class Plan(ctypes.Structure):
    """Mirror of tac_plan (filled by tac_prepare_weights)."""
    _fields_ = [("prepared", ctypes.c_void_p), ("bytes", ctypes.c_size_t),
                ("fingerprint", ctypes.c_uint64), ("abi_version", ctypes.c_int32),
                ("scale_code", ctypes.c_int32)]


class GradDesc(ctypes.Structure):
    """Mirror of tac_grad_desc."""
    _fields_ = [("surrogate", ctypes.c_int32), ("alpha", ctypes.c_float), ("detach_reset", ctypes.c_int32)]


class Prepared:
    """A prepared layer: the device image (torch uint8 tensor, kept alive here) and the
    host tac_plan that names it."""

    def __init__(self, buf: torch.Tensor, plan: Plan):
        self.buf = buf
        self.plan = plan

    @property
    def device(self):
        return self.buf.device


_lock = threading.Lock()
_L = None


def lib():
    """Load libtacsnn.so (built by ``python -m paper_2603_13810_b200.build``)."""
    global _L
    with _lock:
        if _L is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"libtacsnn.so not found at {LIB_PATH}; build it with "
                                   "`python -m paper_2603_13810_b200.build` (no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            P, i32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
            D = ctypes.POINTER(Desc)
            sig = {
                "tac_desc_check": ([D], i32),
                "tac_out_shape": ([D, P, P, P, P], i32),
                "tac_select_engine": ([D], i32),
                "tac_weights_bytes": ([D, ctypes.POINTER(sz)], i32),
                "tac_prepare_weights": ([D, P, P, P, sz, P, ctypes.POINTER(Plan)], i32),
                "tac_workspace_bytes": ([D, ctypes.POINTER(sz)], i32),
                "tac_conv_lif_forward": ([D, ctypes.POINTER(Plan), P, P, P, P, P, P, sz, P], i32),
                "tac_conv_lif_forward_real": ([D, ctypes.POINTER(Plan), P, P, P, P, P, P, sz, P], i32),
                "tac_pack_spikes": ([P, P, i32, i32, i32, i32, i32, P], i32),
                "tac_unpack_spikes": ([P, P, i32, i32, i32, i32, i32, P], i32),
                "tac_status_string": ([i32], ctypes.c_char_p),
                "tac_last_error_detail": ([], ctypes.c_char_p),
                "tac_abi_version": ([], i32),
                "tac_last_launch_count": ([], i32),
                "tac_debug_set_trace": ([P], None),
                "tac_conv_lif_forward_train": ([D, ctypes.POINTER(Plan), P, P, P, P, P, P, P], i32),
                "tac_backward_workspace_bytes": ([D, ctypes.POINTER(sz)], i32),
                "tac_conv_lif_backward": ([D, ctypes.POINTER(Plan), ctypes.POINTER(GradDesc), P, P, P, P, P,
                                           P, P, P, P, P, P, sz, P], i32),
                "tac_or_pool2": ([P, P, i32, i32, i32, i32, i32, P], i32),
                "tac_or_pool2_backward": ([P, P, P, i32, i32, i32, i32, i32, P], i32),
                "tac_vote": ([P, i32, i32, i32, i32, P, P], i32),
            }
            for name, (args, res) in sig.items():
                f = getattr(L, name)
                f.argtypes, f.restype = args, res
            _L = L
    return _L


def _check(status):
    if status != 0:
        L = lib()
        raise RuntimeError(f"{L.tac_status_string(status).decode()}: "
                           f"{L.tac_last_error_detail().decode()}")


@dataclasses.dataclass(frozen=True)
class LayerSpec:
    """One Conv-LIF layer (include/tacsnn.h tac_conv_lif_desc)."""
    T: int
    B: int
    C_in: int
    H: int
    W: int
    C_out: int
    R: int = 3
    S: int = 3
    stride: int = 1
    pad: int = 0
    K: int = 1
    mode: str = "tac"
    beta: float = 0.9
    v_th: float = 1.0
    v_reset: float = 0.0
    reset: str = "subtract"
    out_pool: int = 1
    engine: str = "auto"
    input: str = "spikes"     # "real": continuous-valued fp32 input frames (tac_conv_lif_forward_real)
    partial: bool = False     # K need not divide T: ceil(T/K) groups, the last one short
    agg_weights: tuple | None = None  # learnable aggregation weights alpha_j (K floats)

    def replace(self, **kw) -> "LayerSpec":
        return dataclasses.replace(self, **kw)

    def desc(self, in_strides=(0, 0), out_strides=(0, 0)) -> Desc:
        alpha = None
        if self.agg_weights is not None:
            assert len(self.agg_weights) == self.K, "agg_weights needs K entries"
            alpha = (ctypes.c_float * self.K)(*self.agg_weights)
        d = Desc(self.T, self.B, self.C_in, self.H, self.W, self.C_out, self.R, self.S,
                 self.stride, self.pad, 1 if self.mode == "dense" else self.K,
                 MODES[self.mode], self.beta, self.v_th, self.v_reset, RESETS[self.reset],
                 self.out_pool, ENGINES[self.engine], in_strides[0], in_strides[1],
                 out_strides[0], out_strides[1], INPUTS[self.input], int(self.partial),
                 ctypes.cast(alpha, ctypes.POINTER(ctypes.c_float)) if alpha is not None else None)
        d._alpha_keepalive = alpha
        return d

    @property
    def conv_hw(self):
        return ((self.H + 2 * self.pad - self.R) // self.stride + 1,
                (self.W + 2 * self.pad - self.S) // self.stride + 1)

    @property
    def in_words_per_row(self):
        return (self.W * self.C_in + 31) // 32

    def out_shape(self):
        """(T_out, H_o, W_o, words_per_row) of the packed output."""
        vals = [ctypes.c_int32() for _ in range(4)]
        d = self.desc()
        _check(lib().tac_out_shape(ctypes.byref(d), *[ctypes.byref(v) for v in vals]))
        return tuple(v.value for v in vals)

    def engine_used(self) -> str:
        d = self.desc()
        e = lib().tac_select_engine(ctypes.byref(d))
        if e < 0:
            _check(lib().tac_desc_check(ctypes.byref(d)))
            raise RuntimeError("requested engine cannot run this layer")
        return ENGINE_NAMES[e]

    def check(self):
        d = self.desc()
        _check(lib().tac_desc_check(ctypes.byref(d)))


def _stream(device=None):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def prepare_weights(spec: LayerSpec, weight: torch.Tensor, bias: torch.Tensor | None = None,
                    device="cuda") -> Prepared:
    """Build the device image and its tac_plan (tac_prepare_weights)."""
    d = spec.desc()
    nbytes = ctypes.c_size_t()
    _check(lib().tac_weights_bytes(ctypes.byref(d), ctypes.byref(nbytes)))
    w = weight.detach().to("cpu", torch.float32).contiguous()
    assert tuple(w.shape) == (spec.C_out, spec.C_in, spec.R, spec.S), w.shape
    b = None if bias is None else bias.detach().to("cpu", torch.float32).contiguous()
    buf = torch.empty(nbytes.value + 256, dtype=torch.uint8, device=device)
    off = (-buf.data_ptr()) % 256
    prep = buf[off:off + nbytes.value]
    plan = Plan()
    _check(lib().tac_prepare_weights(ctypes.byref(d), _ptr(w), _ptr(b), _ptr(prep),
                                     nbytes.value, _stream(prep.device), ctypes.byref(plan)))
    return Prepared(prep, plan)


def conv_lif(spec: LayerSpec, prepared: Prepared, x: torch.Tensor, *, v_init=None,
             want_v_final=False, want_counts=True, out: torch.Tensor | None = None,
             workspace: bool = True):
    """Run one layer (tac_conv_lif_forward) on the current stream.

    x: int32/uint32-bit packed spikes [T, B, H, WPR] (rows contiguous; T and B
    strides taken from the tensor), or for spec.input == "real" fp32 frames
    [T, B, H, W, C_in] (tac_conv_lif_forward_real; each (t, b) plane contiguous).
    Returns (spikes_out [T_out,B,H_o,WPR_out] int32, v_final [B,H',W',C_out] fp32 or
    None, counts [B,C_out] int32 or None).
    """
    real = spec.input == "real"
    if real:
        if not (x.is_cuda and x.dtype == torch.float32 and x.dim() == 5):
            raise ValueError("real input: fp32 cuda tensor [T, B, H, W, C_in]")
        if tuple(x.shape) != (spec.T, spec.B, spec.H, spec.W, spec.C_in):
            raise ValueError(f"x shape {tuple(x.shape)} != {(spec.T, spec.B, spec.H, spec.W, spec.C_in)}")
        if not (x.stride(4) == 1 and x.stride(3) == spec.C_in and x.stride(2) == spec.W * spec.C_in):
            raise ValueError("each (t, b) plane of x must be contiguous")
    else:
        if not (x.is_cuda and x.dtype == torch.int32 and x.dim() == 4):
            raise ValueError("spikes: packed int32 cuda tensor [T, B, H, WPR]")
        if tuple(x.shape) != (spec.T, spec.B, spec.H, spec.in_words_per_row):
            raise ValueError(f"x shape {tuple(x.shape)} != {(spec.T, spec.B, spec.H, spec.in_words_per_row)}")
        if not (x.stride(3) == 1 and x.stride(2) == spec.in_words_per_row):
            raise ValueError("rows must be packed")
    T_out, Ho, Wo, wpr = spec.out_shape()
    if out is None:
        out = torch.empty((T_out, spec.B, Ho, wpr), dtype=torch.int32, device=x.device)
    assert tuple(out.shape) == (T_out, spec.B, Ho, wpr) and out.stride(3) == 1 and out.stride(2) == wpr
    hc, wc = spec.conv_hw
    v_final = torch.empty((spec.B, hc, wc, spec.C_out), dtype=torch.float32,
                          device=x.device) if want_v_final else None
    counts = torch.empty((spec.B, spec.C_out), dtype=torch.int32,
                         device=x.device) if want_counts else None
    if v_init is not None:
        assert v_init.is_cuda and v_init.dtype == torch.float32 and v_init.is_contiguous()
        assert tuple(v_init.shape) == (spec.B, hc, wc, spec.C_out)
    d = spec.desc((x.stride(0), x.stride(1)), (out.stride(0), out.stride(1)))
    wsb = ctypes.c_size_t()
    _check(lib().tac_workspace_bytes(ctypes.byref(d), ctypes.byref(wsb)))
    # workspace: required for K not dividing T; optional for two-phase tcgen05 FC layers
    # (workspace=False exercises their fused path -- the library then needs none)
    need_ws = wsb.value and (workspace or (spec.partial and spec.T % spec.K != 0 and spec.mode != "dense"))
    ws = torch.empty(wsb.value, dtype=torch.uint8, device=x.device) if need_ws else None
    fwd = lib().tac_conv_lif_forward_real if real else lib().tac_conv_lif_forward
    _check(fwd(ctypes.byref(d), ctypes.byref(prepared.plan), _ptr(x), _ptr(v_init), _ptr(out), _ptr(v_final),
               _ptr(counts), _ptr(ws), wsb.value if ws is not None else 0, _stream(x.device)))
    return out, v_final, counts


def _check_input(spec: LayerSpec, x: torch.Tensor):
    if spec.input == "real":
        if not (x.is_cuda and x.dtype == torch.float32 and tuple(x.shape) == (spec.T, spec.B, spec.H, spec.W, spec.C_in)):
            raise ValueError("real input: fp32 cuda [T, B, H, W, C_in]")
    elif not (x.is_cuda and x.dtype == torch.int32 and tuple(x.shape) == (spec.T, spec.B, spec.H, spec.in_words_per_row)
              and x.stride(3) == 1 and x.stride(2) == spec.in_words_per_row):
        raise ValueError("spikes: packed int32 cuda [T, B, H, WPR] with packed rows")


def conv_lif_train(spec: LayerSpec, prepared: Prepared, x: torch.Tensor, *, v_init=None,
                   want_v_final=False, want_counts=False):
    """Training forward (tac_conv_lif_forward_train): as conv_lif, plus y_seq, the per-group
    drive fp32 [G, B, H', W', C_out] that conv_lif_backward replays.
    Returns (spikes_out, v_final or None, counts or None, y_seq)."""
    _check_input(spec, x)
    T_out, Ho, Wo, wpr = spec.out_shape()
    hc, wc = spec.conv_hw
    G = spec.T // (1 if spec.mode == "dense" else spec.K)
    out = torch.empty((T_out, spec.B, Ho, wpr), dtype=torch.int32, device=x.device)
    v_final = torch.empty((spec.B, hc, wc, spec.C_out), dtype=torch.float32, device=x.device) if want_v_final else None
    counts = torch.empty((spec.B, spec.C_out), dtype=torch.int32, device=x.device) if want_counts else None
    y_seq = torch.empty((G, spec.B, hc, wc, spec.C_out), dtype=torch.float32, device=x.device)
    d = spec.desc((x.stride(0), x.stride(1)), (out.stride(0), out.stride(1)))
    _check(lib().tac_conv_lif_forward_train(ctypes.byref(d), ctypes.byref(prepared.plan), _ptr(x), _ptr(v_init),
                                            _ptr(out), _ptr(v_final), _ptr(counts), _ptr(y_seq),
                                            _stream(x.device)))
    return out, v_final, counts, y_seq


def conv_lif_backward(spec: LayerSpec, prepared: Prepared, x: torch.Tensor, y_seq: torch.Tensor,
                      g_spikes: torch.Tensor, *, v_init=None, g_v_final=None, surrogate="fast_sigmoid",
                      alpha=25.0, detach_reset=False, want_input_grad=True, want_v_init_grad=False,
                      want_agg_grad=False):
    """Surrogate-gradient BPTT of one layer (tac_conv_lif_backward).  g_spikes: fp32
    [T_out, B, H', W', C_out] = dL/ds.  Returns dict(g_weight [C_out,C_in,R,S], g_bias,
    g_input [T,B,H,W,C_in] or None, g_v_init or None, g_agg_weights or None)."""
    _check_input(spec, x)
    hc, wc = spec.conv_hw
    dev = x.device
    g_w = torch.empty((spec.C_out, spec.C_in, spec.R, spec.S), dtype=torch.float32, device=dev)
    g_b = torch.empty((spec.C_out,), dtype=torch.float32, device=dev)
    g_in = torch.empty((spec.T, spec.B, spec.H, spec.W, spec.C_in), dtype=torch.float32,
                       device=dev) if want_input_grad else None
    g_vi = torch.empty((spec.B, hc, wc, spec.C_out), dtype=torch.float32, device=dev) if want_v_init_grad else None
    g_a = torch.empty((spec.K,), dtype=torch.float32, device=dev) if want_agg_grad else None
    d = spec.desc((x.stride(0), x.stride(1)), (0, 0))
    wsb = ctypes.c_size_t()
    _check(lib().tac_backward_workspace_bytes(ctypes.byref(d), ctypes.byref(wsb)))
    ws = torch.empty(wsb.value, dtype=torch.uint8, device=dev)
    gd = GradDesc(SURROGATES[surrogate], float(alpha), int(bool(detach_reset)))
    _check(lib().tac_conv_lif_backward(ctypes.byref(d), ctypes.byref(prepared.plan), ctypes.byref(gd), _ptr(x),
                                       _ptr(v_init), _ptr(y_seq), _ptr(g_spikes.contiguous()), _ptr(g_v_final),
                                       _ptr(g_w), _ptr(g_b), _ptr(g_in), _ptr(g_vi), _ptr(g_a), _ptr(ws),
                                       wsb.value, _stream(dev)))
    return dict(g_weight=g_w, g_bias=g_b, g_input=g_in, g_v_init=g_vi, g_agg_weights=g_a)


def or_pool2(x: torch.Tensor, C: int, W: int) -> torch.Tensor:
    """2x2 OR-pool of packed spikes [T, B, H, WPR] (tac_or_pool2)."""
    T, B, H, wpr = x.shape
    assert x.is_cuda and x.dtype == torch.int32 and x.is_contiguous() and wpr == (W * C + 31) // 32
    out = torch.empty((T, B, H // 2, ((W // 2) * C + 31) // 32), dtype=torch.int32, device=x.device)
    _check(lib().tac_or_pool2(_ptr(x), _ptr(out), T, B, C, H, W, _stream(x.device)))
    return out


def or_pool2_backward(pre: torch.Tensor, g_pooled: torch.Tensor, C: int, W: int) -> torch.Tensor:
    """MaxPool2d-semantics backward of or_pool2: g_pooled fp32 [T, B, H/2, W/2, C] ->
    fp32 [T, B, H, W, C] (tac_or_pool2_backward)."""
    T, B, H, _ = pre.shape
    g = torch.empty((T, B, H, W, C), dtype=torch.float32, device=pre.device)
    _check(lib().tac_or_pool2_backward(_ptr(pre.contiguous()), _ptr(g_pooled.contiguous()), _ptr(g), T, B, C, H,
                                       W, _stream(pre.device)))
    return g


def vote(counts: torch.Tensor, voters: int, T_out: int) -> torch.Tensor:
    """VotingLayer (tac_vote): counts int32 [B, C] -> fp32 class scores [B, C // voters],
    the mean firing rate of each class's voters."""
    assert counts.is_cuda and counts.dtype == torch.int32 and counts.is_contiguous() and counts.dim() == 2
    B, C = counts.shape
    scores = torch.empty((B, C // voters), dtype=torch.float32, device=counts.device)
    _check(lib().tac_vote(_ptr(counts), B, C, voters, T_out, _ptr(scores), _stream(counts.device)))
    return scores


def pack(dense: torch.Tensor) -> torch.Tensor:
    """u8 {0,1} [T,B,C,H,W] (cuda) -> packed int32 [T,B,H,WPR] (tac_pack_spikes)."""
    assert dense.is_cuda and dense.dtype == torch.uint8 and dense.is_contiguous()
    T, B, C, H, W = dense.shape
    out = torch.empty((T, B, H, (W * C + 31) // 32), dtype=torch.int32, device=dense.device)
    _check(lib().tac_pack_spikes(_ptr(dense), _ptr(out), T, B, C, H, W, _stream(dense.device)))
    return out


def unpack(packed: torch.Tensor, C: int, W: int) -> torch.Tensor:
    """packed int32 [T,B,H,WPR] (cuda, contiguous) -> u8 [T,B,C,H,W] (tac_unpack_spikes)."""
    assert packed.is_cuda and packed.dtype == torch.int32 and packed.is_contiguous()
    T, B, H, wpr = packed.shape
    assert wpr == (W * C + 31) // 32
    out = torch.empty((T, B, C, H, W), dtype=torch.uint8, device=packed.device)
    _check(lib().tac_unpack_spikes(_ptr(packed), _ptr(out), T, B, C, H, W,
                                   _stream(packed.device)))
    return out


def last_launch_count() -> int:
    return int(lib().tac_last_launch_count())


def abi_version() -> int:
    return int(lib().tac_abi_version())
