"""ctypes binding of include/lp.h (argument marshalling only).

Loads the in-tree liblp_b200.so. There is no fallback: if the library is
missing or fails to load, import raises. Every step of the hot path runs in
the library's CUDA kernels.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LP_LIB_PATH") or os.path.join(_HERE, "liblp_b200.so")  # override: A/B builds only

LP_OK, LP_ERR_INVALID_ARG, LP_ERR_UNSUPPORTED, LP_ERR_MISALIGNED, LP_ERR_CUDA = range(5)
LP_GRID_TRIPLANE, LP_GRID_VOXEL = 0, 1
LP_CONTRACT_NONE, LP_CONTRACT_PER_AXIS, LP_CONTRACT_RADIAL = 0, 1, 2
LP_ABI_VERSION = 3
LP_MAX_LAYERS = 8
_STATUS = {0: "LP_OK", 1: "LP_ERR_INVALID_ARG", 2: "LP_ERR_UNSUPPORTED", 3: "LP_ERR_MISALIGNED", 4: "LP_ERR_CUDA"}

# Every symbol include/lp.h declares (tests check the library exports them all).
EXPORTED = ("lp_render_forward", "lp_render_backward", "lp_fwd_bwd_host_workspace_bytes",
            "lp_render_fwd_bwd_host", "lp_splat_forward", "lp_splat_normalize", "lp_splat_backward",
            "lp_splat_forward_mlp", "lp_splat_backward_mlp",
            "lp_set_l2_persist", "lp_last_error", "lp_abi_version")


class LpGrid(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("H", ctypes.c_int32), ("W", ctypes.c_int32), ("D", ctypes.c_int32),
                ("K", ctypes.c_int32), ("data", ctypes.c_void_p * 3), ("contraction", ctypes.c_int32),
                ("contract_scale", ctypes.c_float)]


class LpMlp(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("widths", ctypes.c_int32 * (LP_MAX_LAYERS + 1)),
                ("params", ctypes.c_void_p), ("dir_freqs", ctypes.c_int32)]


class LpRays(ctypes.Structure):
    _fields_ = [("n_rays", ctypes.c_int64), ("origins", ctypes.c_void_p), ("dirs", ctypes.c_void_p),
                ("t_near", ctypes.c_void_p), ("t_far", ctypes.c_void_p), ("n_samples", ctypes.c_int32)]


class LpSplatMlp(ctypes.Structure):
    _fields_ = [("params", ctypes.c_void_p), ("hidden", ctypes.c_int32), ("C_in", ctypes.c_int32),
                ("dir_freqs", ctypes.c_int32), ("K_prior", ctypes.c_int32), ("prior", ctypes.c_void_p * 3),
                ("n_hidden", ctypes.c_int32)]


class LpError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2404_19760_b200/build.py` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    gp, mp, rp = ctypes.POINTER(LpGrid), ctypes.POINTER(LpMlp), ctypes.POINTER(LpRays)
    L.lp_render_forward.argtypes = [gp, mp, rp, P, P, P, P, P]
    L.lp_render_backward.argtypes = [gp, mp, rp, P, P, P, P, P, ctypes.POINTER(ctypes.c_void_p), P, P]
    L.lp_fwd_bwd_host_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int32]
    L.lp_fwd_bwd_host_workspace_bytes.restype = ctypes.c_size_t
    L.lp_render_fwd_bwd_host.argtypes = [gp, mp, rp, P, P, P, P, P, ctypes.POINTER(ctypes.c_void_p), P, P,
                                         ctypes.c_size_t, P]
    P3 = ctypes.POINTER(ctypes.c_void_p)
    L.lp_splat_forward.argtypes = [gp, rp, P, P3, P3, P]
    L.lp_splat_normalize.argtypes = [gp, P3, P3, P3, P]
    L.lp_splat_backward.argtypes = [gp, rp, P3, P3, P, P]
    sp = ctypes.POINTER(LpSplatMlp)
    L.lp_splat_forward_mlp.argtypes = [gp, rp, P, sp, P3, P3, P]
    L.lp_splat_backward_mlp.argtypes = [gp, rp, P, sp, P3, P3, P, P3, P, P]
    L.lp_set_l2_persist.argtypes = [ctypes.c_float]
    L.lp_last_error.restype = ctypes.c_char_p
    for f in (L.lp_render_forward, L.lp_render_backward, L.lp_render_fwd_bwd_host, L.lp_set_l2_persist,
              L.lp_abi_version, L.lp_splat_forward, L.lp_splat_normalize, L.lp_splat_backward,
              L.lp_splat_forward_mlp, L.lp_splat_backward_mlp):
        f.restype = ctypes.c_int
    if L.lp_abi_version() != LP_ABI_VERSION:
        raise ImportError(f"{LIB_PATH} has ABI {L.lp_abi_version()}, expected {LP_ABI_VERSION}: rebuild it")
    return L


lib = _load()


def check(status: int):
    if status != LP_OK:
        raise LpError(status, lib.lp_last_error().decode())


def make_grid(kind: int, H: int, W: int, D: int, K: int, ptrs, contraction: int = 0,
              contract_scale: float = 1.0) -> LpGrid:
    g = LpGrid()
    g.kind, g.H, g.W, g.D, g.K = kind, H, W, D, K
    g.contraction, g.contract_scale = int(contraction), float(contract_scale)
    for i in range(3):
        g.data[i] = ptrs[i] if i < len(ptrs) else None
    return g


def make_mlp(widths, params_ptr, dir_freqs: int = 0) -> LpMlp:
    m = LpMlp()
    m.dir_freqs = int(dir_freqs)
    m.n_layers = len(widths) - 1
    for i, w in enumerate(widths):
        m.widths[i] = int(w)
    m.params = params_ptr
    return m


def make_rays(n: int, o, d, near, far, S: int) -> LpRays:
    r = LpRays()
    r.n_rays, r.origins, r.dirs, r.t_near, r.t_far, r.n_samples = n, o, d, near, far, S
    return r


def ptr_array3(ptrs):
    arr = (ctypes.c_void_p * 3)()
    for i in range(3):
        arr[i] = ptrs[i] if i < len(ptrs) else None
    return arr
