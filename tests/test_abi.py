"""The C-ABI library loads, exports every symbol include/lp.h declares, and
rejects bad arguments host-side before any CUDA call (no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "lp.h")).read()
    return sorted(set(re.findall(r"^\s*(?:lp_status|size_t|const char\*|int)\s+(lp_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def L():
    from paper_2404_19760_b200 import _lib
    return _lib


def test_library_exports_every_declared_symbol(L):
    declared = _declared_symbols()
    assert len(declared) >= 7
    for name in declared:
        assert hasattr(L.lib, name), name
    assert set(declared) == set(L.EXPORTED)
    assert L.lib.lp_abi_version() == L.LP_ABI_VERSION == 3


def _args(L, K=8, widths=(8, 16, 4), kind=0, ptr=0x1000, S=8, n=4):
    g = L.make_grid(kind, 4, 4, 4, K, [ptr, ptr, ptr])
    m = L.make_mlp(widths, ptr)
    r = L.make_rays(n, ptr, ptr, ptr, ptr, S)
    return g, m, r


def _fwd(L, g, m, r):
    p = ctypes.c_void_p(0x2000)
    return L.lib.lp_render_forward(ctypes.byref(g), ctypes.byref(m), ctypes.byref(r), None, p, p, None, None)


def test_validation_errors(L):
    g, m, r = _args(L)
    assert L.lib.lp_render_forward(None, ctypes.byref(m), ctypes.byref(r), None, None, None, None, None) == L.LP_ERR_INVALID_ARG
    assert "null" in L.lib.lp_last_error().decode()
    g, m, r = _args(L, S=1)
    assert _fwd(L, g, m, r) == L.LP_ERR_INVALID_ARG
    g, m, r = _args(L, K=12, widths=(12, 16, 4))
    assert _fwd(L, g, m, r) == L.LP_ERR_UNSUPPORTED
    g, m, r = _args(L, widths=(4, 16, 4))
    assert _fwd(L, g, m, r) == L.LP_ERR_INVALID_ARG
    g, m, r = _args(L, ptr=0x1004)
    assert _fwd(L, g, m, r) == L.LP_ERR_MISALIGNED
    g, m, r = _args(L, kind=5)
    assert _fwd(L, g, m, r) == L.LP_ERR_INVALID_ARG
    g, m, r = _args(L, widths=(8, 16, 32, 4))      # 3 layers with mismatched hidden widths
    assert _fwd(L, g, m, r) == L.LP_ERR_UNSUPPORTED
    assert L.lib.lp_set_l2_persist(ctypes.c_float(2.0)) == L.LP_ERR_INVALID_ARG
    g, m, r = _args(L)
    g.contraction = 3                              # unknown contraction mode
    assert _fwd(L, g, m, r) == L.LP_ERR_INVALID_ARG
    g.contraction, g.contract_scale = L.LP_CONTRACT_PER_AXIS, 2.5   # scale a outside (0, 2)
    assert _fwd(L, g, m, r) == L.LP_ERR_INVALID_ARG and "contract_scale" in L.lib.lp_last_error().decode()


def test_workspace_size(L):
    n = L.lib.lp_fwd_bwd_host_workspace_bytes(1000, 3)
    assert n >= 1000 * (12 + 12 + 4 + 4 + 12 + 12 + 4 + 4)


def test_fwd_bwd_host_validates_before_enqueue(L):
    """lp_render_fwd_bwd_host rejects null gradient buffers, a short or
    misaligned workspace and null host buffers host-side (no CUDA call)."""
    g, m, r = _args(L)
    p = ctypes.c_void_p(0x2000)
    need = L.lib.lp_fwd_bwd_host_workspace_bytes(4, 3)
    ws = ctypes.c_void_p(0x10000)
    gptr = L.ptr_array3([0x4000, 0x4000, 0x4000])
    f = L.lib.lp_render_fwd_bwd_host
    call = lambda gd, gp, w, n, outh: f(ctypes.byref(g), ctypes.byref(m), ctypes.byref(r), None, p, None, outh, p,
                                       gd, gp, w, ctypes.c_size_t(n), None)
    assert call(None, p, ws, need, p) == L.LP_ERR_INVALID_ARG
    assert call(L.ptr_array3([0x4004, 0x4000, 0x4000]), p, ws, need, p) == L.LP_ERR_MISALIGNED
    assert call(gptr, None, ws, need, p) == L.LP_ERR_INVALID_ARG
    assert call(gptr, p, ws, need - 1, p) == L.LP_ERR_INVALID_ARG
    assert call(gptr, p, ctypes.c_void_p(0x10010), need, p) == L.LP_ERR_MISALIGNED
    assert call(gptr, p, ws, need, None) == L.LP_ERR_INVALID_ARG
    g.contraction, g.contract_scale = L.LP_CONTRACT_PER_AXIS, 2.0   # a = 2 collapses the background: rejected
    assert call(gptr, p, ws, need, p) == L.LP_ERR_INVALID_ARG


def test_splat_mlp_descriptor_validation(L):
    """lp_splat_forward_mlp rejects g_s descriptors no kernel is compiled for
    (hidden width, channel counts, n_hidden outside {1, 2}) before any CUDA call;
    n_hidden = 0 reads as 1 (ABI 2 callers zero-initialise it)."""
    g = L.make_grid(1, 4, 4, 4, 32, [0x1000, 0x1000, 0x1000])
    r = L.make_rays(4, 0x1000, 0x1000, 0x1000, 0x1000, 8)
    P3 = L.ptr_array3([0x1000, 0x1000, 0x1000])

    def gs(**kw):
        m = L.LpSplatMlp()
        m.params, m.hidden, m.C_in, m.dir_freqs, m.K_prior, m.n_hidden = 0x1000, 64, 32, 4, 32, 1
        for k, v in kw.items():
            setattr(m, k, v)
        for i in range(3):
            m.prior[i] = 0x1000
        return m
    call = lambda m: L.lib.lp_splat_forward_mlp(ctypes.byref(g), ctypes.byref(r), ctypes.c_void_p(0x1000),
                                                ctypes.byref(m), P3, P3, None)
    assert call(gs(n_hidden=3)) == L.LP_ERR_UNSUPPORTED and "n_hidden" in L.lib.lp_last_error().decode()
    assert call(gs(n_hidden=-1)) == L.LP_ERR_UNSUPPORTED
    assert call(gs(hidden=32)) == L.LP_ERR_UNSUPPORTED
    assert call(gs(C_in=16, n_hidden=2)) == L.LP_ERR_UNSUPPORTED
    assert call(gs(dir_freqs=6)) == L.LP_ERR_INVALID_ARG
