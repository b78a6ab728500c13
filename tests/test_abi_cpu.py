"""CPU-only checks of the C ABI boundary: the library builds and loads, exports
every function include/tacsnn.h declares, and its host-side validation returns
the documented statuses (no device call is made by these functions)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def T():
    from paper_2603_13810_b200 import build, tacsnn
    build.build()
    return tacsnn


def _declared_functions():
    with open(os.path.join(ROOT, "include", "tacsnn.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tac_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(T):
    L = T.lib()
    decl = _declared_functions()
    assert len(decl) >= 13
    for name in decl:
        assert hasattr(L, name), f"{name} declared in include/tacsnn.h but not exported"
    assert set(decl) == set(T.EXPORTS)
    assert T.abi_version() == T.ABI_VERSION == 3


def test_status_strings(T):
    L = T.lib()
    for code, name in enumerate(["TAC_OK", "TAC_ERR_NULL", "TAC_ERR_SHAPE",
                                 "TAC_ERR_K_NOT_DIVIDING_T", "TAC_ERR_PARAM",
                                 "TAC_ERR_NONFINITE", "TAC_ERR_ALIGN", "TAC_ERR_UNSUPPORTED",
                                 "TAC_ERR_WORKSPACE", "TAC_ERR_CUDA"]):
        assert L.tac_status_string(code).decode() == name


def _status(T, spec):
    d = spec.desc()
    return T.lib().tac_desc_check(ctypes.byref(d)), T.lib().tac_last_error_detail().decode()


def test_validation_statuses(T):
    base = T.LayerSpec(T=16, B=4, C_in=2, H=32, W=32, C_out=16, pad=1, K=4, mode="tactp", beta=0.5)
    assert _status(T, base)[0] == 0
    st, detail = _status(T, base.replace(K=3))
    assert st == 3 and "K=3" in detail                      # K does not divide T
    assert _status(T, base.replace(K=0))[0] == 3
    assert _status(T, base.replace(K=3, partial=True))[0] == 0      # opt-in short last group
    assert _status(T, base.replace(mode="dense", K=3))[0] == 0   # K ignored for dense
    assert _status(T, base.replace(beta=1.0))[0] == 4
    assert _status(T, base.replace(beta=0.0))[0] == 4
    assert _status(T, base.replace(v_th=0.0))[0] == 4
    assert _status(T, base.replace(beta=float("nan")))[0] == 5
    assert _status(T, base.replace(v_reset=float("inf")))[0] == 5
    assert _status(T, base.replace(H=0))[0] == 2
    assert _status(T, base.replace(H=1, pad=0))[0] == 2         # H' < 1
    assert _status(T, base.replace(out_pool=3))[0] == 4
    assert _status(T, base.replace(W=31, out_pool=2))[0] == 0   # odd extent: floor pooling
    assert base.replace(W=31, out_pool=2).out_shape()[2] == 15
    assert _status(T, base.replace(W=3, pad=0, out_pool=2))[0] == 2   # W' = 1: nothing to pool
    assert _status(T, base.replace(T=64, K=64))[0] == 7         # K > 32
    d = base.desc()
    assert T.lib().tac_desc_check(None) == 1


def test_out_shape(T):
    s = T.LayerSpec(T=32, B=8, C_in=2, H=128, W=128, C_out=128, pad=1, K=4, mode="tactp",
                    beta=0.5, out_pool=2)
    assert s.out_shape() == (32, 64, 64, 64 * 128 // 32)
    assert s.replace(mode="tac").out_shape()[0] == 8
    m = T.LayerSpec(T=16, B=4, C_in=1, H=28, W=28, C_out=32, pad=0, K=4, mode="tac")
    assert m.out_shape() == (4, 26, 26, 26)
    assert m.replace(out_pool=2).out_shape() == (4, 13, 13, 13)


def test_weights_bytes_and_engine_selection(T):
    s = T.LayerSpec(T=8, B=4, C_in=1, H=28, W=28, C_out=8, K=4, mode="tac", beta=0.9)
    n = ctypes.c_size_t()
    d = s.desc()
    assert T.lib().tac_weights_bytes(ctypes.byref(d), ctypes.byref(n)) == 0
    assert n.value >= 8 * 9 * 4 + 8 * 4 and n.value % 256 == 0
    assert s.replace(engine="simt").engine_used() == "simt"
    assert s.engine_used() in ("simt", "tcgen05")
