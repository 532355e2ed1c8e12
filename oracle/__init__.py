"""CPU oracle for the Lightplane Renderer hot path -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package. The product package
(paper_2404_19760_b200) never imports, links or executes it, and this package
never imports the product package: the two share no code. The only shared
module is `workload` (seeded input generators, no method arithmetic).

The arithmetic lives in lp_oracle.cpp (plain fp64 C++, per-ray store-all
forward of Eq. 1 and hand-derived backward of Eq. 3; see its header for the
paper citations). This file only compiles it and marshals numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lp_oracle.cpp")
_LIB = os.path.join(_HERE, "liblp_oracle.so")
_lib = None
_lock = threading.Lock()

TRIPLANE = 0
VOXEL = 1


def build(force: bool = False) -> str:
    """Compile lp_oracle.cpp into liblp_oracle.so (g++ -O3, fp64, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-shared", "-fno-fast-math",
               "-ffp-contract=off", _SRC, "-o", tmp]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i32, i64, f64 = ctypes.c_int, ctypes.c_int64, ctypes.c_double
            L.lpo_sample.argtypes = [i32, i32, i32, i32, i32, P, P, P, i64, P, P]
            L.lpo_splat.argtypes = [i32, i32, i32, i32, i32, i64, P, P, P, P, P]
            L.lpo_mlp_forward.argtypes = [i32, P, P, i64, P, P]
            L.lpo_mlp_backward.argtypes = [i32, P, P, i64, P, P, P, P]
            L.lpo_render_forward.argtypes = [i32, i32, i32, i32, i32, P, P, P, i32, P, P, i64, i64,
                                             P, P, P, P, i32, P, P, P, P, i32, f64, i32]
            L.lpo_render_backward.argtypes = [i32, i32, i32, i32, i32, P, P, P, i32, P, P, i64, i64,
                                              P, P, P, P, i32, P, P, P, P, P, P, P, i32, P, i32, f64, i32]
            L.lpo_trace.argtypes = [i32, i32, i32, i32, i32, P, P, P, i32, P, P, P, P, f64, f64, i32,
                                    P, P, P, P, P, i32, f64, i32]
            L.lpo_render_relu_slack.argtypes = [i32, i32, i32, i32, i32, P, P, P, i32, P, P, i64, i64,
                                                P, P, P, P, i32, P, P, P, f64, P, P, P, P, P, i32, f64, i32]
            L.lpo_contract.argtypes = [i32, f64, i64, P, P]
            L.lpo_splat_rays.argtypes = [i32, i32, i32, i32, i32, i64, i64, P, P, P, P, i32, P, P, P, P, P, P, P,
                                         i32, f64]
            L.lpo_splat_normalize.argtypes = [i64, i32, P, P, P]
            L.lpo_splat_rays_mlp.argtypes = [i32, i32, i32, i32, i32, i32, P, P, P, i32, P, P, i32, i32, i64, i64,
                                             P, P, P, P, i32, P, P, P, P, P, P, P, i32, f64]
            L.lpo_splat_mlp_relu_slack.argtypes = [i32, i32, i32, i32, i32, i32, P, P, P, i32, P, P, i32, i32, i64,
                                                   i64, P, P, P, P, i32, P, P, P, P, P, P, P, f64, P, P, P, P, P,
                                                   i32, f64]
            L.lpo_splat_rays_mlp_backward.argtypes = [i32, i32, i32, i32, i32, i32, P, P, P, i32, P, P, i32, i32,
                                                      i64, i64, P, P, P, P, i32, P, P, P, P, P, P, P, P, P, P, P,
                                                      P, i32, f64]
            L.lpo_splat_rays_backward.argtypes = [i32, i32, i32, i32, i32, i64, i64, P, P, P, P, i32, P, P, P,
                                                  P, P, P, P, i32, f64]
            for f in (L.lpo_render_relu_slack, L.lpo_sample, L.lpo_splat, L.lpo_mlp_forward, L.lpo_mlp_backward,
                      L.lpo_render_forward, L.lpo_render_backward, L.lpo_trace, L.lpo_contract,
                      L.lpo_splat_rays, L.lpo_splat_normalize, L.lpo_splat_rays_backward,
                      L.lpo_splat_rays_mlp, L.lpo_splat_rays_mlp_backward, L.lpo_splat_mlp_relu_slack):
                f.restype = ctypes.c_int
            _lib = L
    return _lib


def _d(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class Field:
    """theta (list of planes or one voxel volume, channel-last) + packed MLP,
    plus the scene contraction applied to sample points (0 none, 1 per-axis,
    2 radial; scale a) -- lp_oracle.cpp contract(). dir_freqs = F > 0 makes the
    field view-dependent: params hold g_sigma (widths with output 1) then g_v
    (input K + 6F, output C) -- lp_oracle.cpp split_nets()."""

    def __init__(self, kind: int, grid: Sequence[np.ndarray], widths: Sequence[int], params: np.ndarray,
                 contraction: int = 0, contract_a: float = 1.0, dir_freqs: int = 0):
        self.kind = int(kind)
        self.dir_freqs = int(dir_freqs)
        self.contraction = int(contraction)
        self.contract_a = float(contract_a)
        self.grid = [_d(g) for g in grid]
        if self.kind == TRIPLANE:
            assert len(self.grid) == 3
            H, W, K = self.grid[0].shape
            D = self.grid[1].shape[1]
            assert self.grid[1].shape == (W, D, K) and self.grid[2].shape == (D, H, K)
        else:
            assert len(self.grid) == 1
            H, W, D, K = self.grid[0].shape
        self.H, self.W, self.D, self.K = int(H), int(W), int(D), int(K)
        self.widths = np.ascontiguousarray(np.asarray(widths, dtype=np.int32))
        self.n_layers = len(widths) - 1
        self.params = _d(params)
        self.C = int(widths[-1]) - 1
        assert self.widths[0] == self.K

    def _planes(self):
        g = self.grid + [None] * (3 - len(self.grid))
        return [_p(x) for x in g]

    def _geom(self):
        return (self.kind, self.H, self.W, self.D, self.K)

    def _scene(self):
        return (self.contraction, self.contract_a, self.dir_freqs)


def contract(contraction: int, a: float, x: np.ndarray) -> np.ndarray:
    """CC(x) (Supp. Eq. contract) for points x[n][3]."""
    x = _d(x).reshape(-1, 3)
    out = np.zeros_like(x)
    rc = lib().lpo_contract(int(contraction), float(a), len(x), _p(x), _p(out))
    assert rc == 0
    return out


def sample(field: Field, x: np.ndarray) -> np.ndarray:
    x = _d(x).reshape(-1, 3)
    h = np.zeros((len(x), field.K))
    rc = lib().lpo_sample(*field._geom(), *field._planes(), len(x), _p(x), _p(h))
    assert rc == 0
    return h


def splat(field: Field, x: np.ndarray, v: np.ndarray):
    x = _d(x).reshape(-1, 3)
    v = _d(v).reshape(len(x), field.K)
    g = [np.zeros_like(a) for a in field.grid]
    gp = [_p(a) for a in g] + [None] * (3 - len(g))
    rc = lib().lpo_splat(*field._geom(), len(x), _p(x), _p(v), *gp)
    assert rc == 0
    return g


def mlp_forward(widths, params, x):
    widths = np.ascontiguousarray(np.asarray(widths, dtype=np.int32))
    x = _d(x).reshape(-1, widths[0])
    params = _d(params)
    out = np.zeros((len(x), int(widths[-1])))
    rc = lib().lpo_mlp_forward(len(widths) - 1, _p(widths), _p(params), len(x), _p(x), _p(out))
    assert rc == 0
    return out


def mlp_backward(widths, params, x, dout):
    widths = np.ascontiguousarray(np.asarray(widths, dtype=np.int32))
    x = _d(x).reshape(-1, widths[0])
    dout = _d(dout).reshape(len(x), int(widths[-1]))
    params = _d(params)
    gp = np.zeros_like(params)
    gin = np.zeros_like(x)
    rc = lib().lpo_mlp_backward(len(widths) - 1, _p(widths), _p(params), len(x), _p(x), _p(dout),
                                _p(gp), _p(gin))
    assert rc == 0
    return gp, gin


class Rays:
    def __init__(self, origins, dirs, near, far, S: int):
        self.o = _d(origins).reshape(-1, 3)
        self.d = _d(dirs).reshape(-1, 3)
        self.near = _d(near).reshape(-1)
        self.far = _d(far).reshape(-1)
        self.S = int(S)
        self.n = len(self.o)


def render_forward(field: Field, rays: Rays, bg=None, r0: int = 0, r1: Optional[int] = None,
                   out=None, tau=None, depth=None, return_depth: bool = False):
    """Returns (out [n][C], tau [n]) and, with return_depth / a depth buffer, depth [n]."""
    r1 = rays.n if r1 is None else r1
    if out is None:
        out = np.zeros((rays.n, field.C))
    if tau is None:
        tau = np.zeros(rays.n)
    if return_depth and depth is None:
        depth = np.zeros(rays.n)
    bgd = None if bg is None else _d(bg)
    rc = lib().lpo_render_forward(*field._geom(), *field._planes(), field.n_layers, _p(field.widths),
                                  _p(field.params), r0, r1, _p(rays.o), _p(rays.d), _p(rays.near),
                                  _p(rays.far), rays.S, _p(bgd), _p(out), _p(tau), _p(depth), *field._scene())
    assert rc == 0
    return (out, tau) if depth is None else (out, tau, depth)


def render_backward(field: Field, rays: Rays, grad_out, grad_tau=None, bg=None, mode: int = 0,
                    r0: int = 0, r1: Optional[int] = None, grads=None, grad_depth=None):
    """Returns (grad_grid list, grad_params); accumulates into `grads` if given."""
    r1 = rays.n if r1 is None else r1
    go = _d(grad_out).reshape(rays.n, field.C)
    gt = None if grad_tau is None else _d(grad_tau).reshape(rays.n)
    gd = None if grad_depth is None else _d(grad_depth).reshape(rays.n)
    bgd = None if bg is None else _d(bg)
    if grads is None:
        grads = ([np.zeros_like(a) for a in field.grid], np.zeros_like(field.params))
    gg, gpar = grads
    gp = [_p(a) for a in gg] + [None] * (3 - len(gg))
    rc = lib().lpo_render_backward(*field._geom(), *field._planes(), field.n_layers, _p(field.widths),
                                   _p(field.params), r0, r1, _p(rays.o), _p(rays.d), _p(rays.near),
                                   _p(rays.far), rays.S, _p(bgd), _p(go), _p(gt), *gp, _p(gpar), mode, _p(gd),
                                   *field._scene())
    assert rc == 0
    return gg, gpar


def relu_slack(field: Field, rays: Rays, grad_out, grad_tau=None, bg=None, band: float = 2e-5,
               r0: int = 0, r1: Optional[int] = None, out=None, grad_depth=None):
    """Elementwise bound of how much the gradients may change when any ReLU
    decision with |z| < band * scale is taken the other way (lp_oracle.cpp
    mlp_slack). Returns (slack_grid list, slack_params)."""
    r1 = rays.n if r1 is None else r1
    go = _d(grad_out).reshape(rays.n, field.C)
    gt = None if grad_tau is None else _d(grad_tau).reshape(rays.n)
    gd = None if grad_depth is None else _d(grad_depth).reshape(rays.n)
    bgd = None if bg is None else _d(bg)
    if out is None:
        out = ([np.zeros_like(a) for a in field.grid], np.zeros_like(field.params))
    sg, sp = out
    ptrs = [_p(a) for a in sg] + [None] * (3 - len(sg))
    rc = lib().lpo_render_relu_slack(*field._geom(), *field._planes(), field.n_layers, _p(field.widths),
                                     _p(field.params), r0, r1, _p(rays.o), _p(rays.d), _p(rays.near),
                                     _p(rays.far), rays.S, _p(bgd), _p(go), _p(gt), float(band), *ptrs, _p(sp),
                                     _p(gd), *field._scene())
    assert rc == 0
    return sg, sp


def relu_slack_threaded(field: Field, rays: Rays, grad_out, grad_tau=None, bg=None, band: float = 2e-5,
                        threads: int = 1, grad_depth=None):
    bounds = np.linspace(0, rays.n, threads + 1).astype(np.int64)
    parts = [([np.zeros_like(a) for a in field.grid], np.zeros_like(field.params)) for _ in range(threads)]
    ts = [threading.Thread(target=relu_slack, kwargs=dict(field=field, rays=rays, grad_out=grad_out,
                                                          grad_tau=grad_tau, bg=bg, band=band, r0=int(bounds[i]),
                                                          r1=int(bounds[i + 1]), out=parts[i],
                                                          grad_depth=grad_depth))
          for i in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return [sum(p[0][k] for p in parts) for k in range(len(field.grid))], sum(p[1] for p in parts)


def trace(field: Field, origin, direction, near: float, far: float, S: int):
    """Per-sample (sigma, tau, T, w, c) of one ray (store-all forward)."""
    o = _d(origin).reshape(3)
    d = _d(direction).reshape(3)
    sigma, tau, T, w = (np.zeros(S) for _ in range(4))
    c = np.zeros((S, field.C))
    rc = lib().lpo_trace(*field._geom(), *field._planes(), field.n_layers, _p(field.widths),
                         _p(field.params), _p(o), _p(d), float(near), float(far), S, _p(sigma), _p(tau),
                         _p(T), _p(w), _p(c), *field._scene())
    assert rc == 0
    return sigma, tau, T, w, c


def render_forward_threaded(field: Field, rays: Rays, bg=None, threads: int = 1, return_depth: bool = False):
    """Forward over disjoint contiguous ray ranges on `threads` host threads
    (ctypes releases the GIL)."""
    out = np.zeros((rays.n, field.C))
    tau = np.zeros(rays.n)
    depth = np.zeros(rays.n) if return_depth else None
    bounds = np.linspace(0, rays.n, threads + 1).astype(np.int64)
    ts = [threading.Thread(target=render_forward, args=(field, rays, bg, int(bounds[i]), int(bounds[i + 1]),
                                                        out, tau, depth)) for i in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return (out, tau) if depth is None else (out, tau, depth)


def backward_buffers(field: Field, threads: int):
    """Per-thread private fp64 gradient buffers ([grid planes], params) for
    render_backward_threaded(parts=...)."""
    return [([np.zeros_like(a) for a in field.grid], np.zeros_like(field.params)) for _ in range(threads)]


def render_backward_threaded(field: Field, rays: Rays, grad_out, grad_tau=None, bg=None, threads: int = 1,
                             grad_depth=None, parts=None):
    """Backward with per-thread private gradient buffers, summed in thread order.
    With `parts` (backward_buffers(field, threads), caller-owned) the gradients
    accumulate into those buffers and nothing is summed or returned (timing
    loops: no per-call allocation of grid-sized buffers)."""
    bounds = np.linspace(0, rays.n, threads + 1).astype(np.int64)
    keep = parts is not None
    if not keep:
        parts = backward_buffers(field, threads)
    assert len(parts) == threads
    ts = [threading.Thread(target=render_backward,
                           kwargs=dict(field=field, rays=rays, grad_out=grad_out, grad_tau=grad_tau, bg=bg,
                                       r0=int(bounds[i]), r1=int(bounds[i + 1]), grads=parts[i],
                                       grad_depth=grad_depth))
          for i in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if keep:
        return None
    gg = [sum(p[0][k] for p in parts) for k in range(len(field.grid))]
    gp = sum(p[1] for p in parts)
    return gg, gp


# ---------------------------------------------------------------- Splatter
class GridSpec:
    """Shape of a splat target: kind, (H, W, D), K channels, scene contraction."""

    def __init__(self, kind: int, dims, K: int, contraction: int = 0, contract_a: float = 1.0):
        self.kind, self.K = int(kind), int(K)
        self.H, self.W, self.D = (int(v) for v in dims)
        self.contraction, self.contract_a = int(contraction), float(contract_a)

    def shapes(self, K=None):
        K = self.K if K is None else K
        H, W, D = self.H, self.W, self.D
        return [(H, W, K), (W, D, K), (D, H, K)] if self.kind == TRIPLANE else [(H, W, D, K)]

    def _geom(self, K=None):
        return (self.kind, self.H, self.W, self.D, self.K if K is None else K)


def _ptr3(arrs):
    return [_p(a) for a in arrs] + [None] * (3 - len(arrs))


def splat_rays(spec: GridSpec, rays: Rays, features, r0: int = 0, r1: Optional[int] = None, acc=None):
    """Unnormalised splat of the rays' features and of the weights: returns
    (theta list, theta_weight list), accumulating into `acc` if given."""
    r1 = rays.n if r1 is None else r1
    v = _d(features).reshape(rays.n, spec.K)
    if acc is None:
        acc = ([np.zeros(s) for s in spec.shapes()], [np.zeros(s) for s in spec.shapes(1)])
    th, wt = acc
    rc = lib().lpo_splat_rays(*spec._geom(), r0, r1, _p(rays.o), _p(rays.d), _p(rays.near), _p(rays.far),
                              rays.S, _p(v), *_ptr3(th), *_ptr3(wt), spec.contraction, spec.contract_a)
    assert rc == 0
    return th, wt


def splat_normalize(theta, theta_weight):
    out = []
    for t, w in zip(theta, theta_weight):
        o = np.zeros_like(t)
        rc = lib().lpo_splat_normalize(int(w.size), int(t.shape[-1]), _p(_d(t)), _p(_d(w)), _p(o))
        assert rc == 0
        out.append(o)
    return out


def splat_forward(spec: GridSpec, rays: Rays, features, threads: int = 1):
    """Splatter forward: (normalised theta, theta, theta_weight)."""
    bounds = np.linspace(0, rays.n, threads + 1).astype(np.int64)
    parts = [([np.zeros(s) for s in spec.shapes()], [np.zeros(s) for s in spec.shapes(1)]) for _ in range(threads)]
    ts = [threading.Thread(target=splat_rays, args=(spec, rays, features, int(bounds[i]), int(bounds[i + 1]),
                                                    parts[i])) for i in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    th = [sum(p[0][k] for p in parts) for k in range(len(parts[0][0]))]
    wt = [sum(p[1][k] for p in parts) for k in range(len(parts[0][1]))]
    return splat_normalize(th, wt), th, wt


def splat_backward(spec: GridSpec, rays: Rays, grad_out, theta_weight, r0: int = 0, r1: Optional[int] = None,
                   out=None):
    """dL/d(features) [n][K] of the normalised splat (theta_weight treated as constant)."""
    r1 = rays.n if r1 is None else r1
    g = [_d(a) for a in grad_out]
    w = [_d(a) for a in theta_weight]
    if out is None:
        out = np.zeros((rays.n, spec.K))
    rc = lib().lpo_splat_rays_backward(*spec._geom(), r0, r1, _p(rays.o), _p(rays.d), _p(rays.near),
                                       _p(rays.far), rays.S, *_ptr3(g), *_ptr3(w), _p(out), spec.contraction,
                                       spec.contract_a)
    assert rc == 0
    return out


def splat_backward_threaded(spec: GridSpec, rays: Rays, grad_out, theta_weight, threads: int = 1):
    out = np.zeros((rays.n, spec.K))
    bounds = np.linspace(0, rays.n, threads + 1).astype(np.int64)
    ts = [threading.Thread(target=splat_backward, args=(spec, rays, grad_out, theta_weight, int(bounds[i]),
                                                        int(bounds[i + 1]), out)) for i in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return out


class SplatMlp:
    """g_s of Eq. 2: prior grid theta^ (same kind/dims as the target,
    K_p channels), MLP widths (C_in + K_p + 6F, hidden..., K) and packed params."""

    def __init__(self, prior: Sequence[np.ndarray], widths: Sequence[int], params, C_in: int, dir_freqs: int):
        self.prior = [_d(g) for g in prior]
        self.Kp = int(self.prior[0].shape[-1])
        self.widths = np.ascontiguousarray(np.asarray(widths, dtype=np.int32))
        self.params = _d(params)
        self.C_in, self.F = int(C_in), int(dir_freqs)
        assert self.widths[0] == self.C_in + self.Kp + 6 * self.F

    def _args(self):
        q = _ptr3(self.prior)
        return (self.Kp, *q, len(self.widths) - 1, _p(self.widths), _p(self.params), self.C_in, self.F)


def splat_forward_mlp(spec: GridSpec, rays: Rays, features, g: SplatMlp):
    """Splatter with g_s: (normalised theta, theta, theta_weight)."""
    v = _d(features).reshape(rays.n, g.C_in)
    th = [np.zeros(s) for s in spec.shapes()]
    wt = [np.zeros(s) for s in spec.shapes(1)]
    rc = lib().lpo_splat_rays_mlp(*spec._geom(), *g._args(), 0, rays.n, _p(rays.o), _p(rays.d), _p(rays.near),
                                  _p(rays.far), rays.S, _p(v), *_ptr3(th), *_ptr3(wt), spec.contraction,
                                  spec.contract_a)
    assert rc == 0
    return splat_normalize(th, wt), th, wt


def splat_backward_mlp(spec: GridSpec, rays: Rays, features, g: SplatMlp, grad_out, theta_weight):
    """(dL/d features [n][C_in], dL/d prior planes, dL/d g_s params)."""
    v = _d(features).reshape(rays.n, g.C_in)
    gv = np.zeros((rays.n, g.C_in))
    gpr = [np.zeros_like(a) for a in g.prior]
    gpar = np.zeros_like(g.params)
    go = [_d(a) for a in grad_out]
    w = [_d(a) for a in theta_weight]
    rc = lib().lpo_splat_rays_mlp_backward(*spec._geom(), *g._args(), 0, rays.n, _p(rays.o), _p(rays.d),
                                           _p(rays.near), _p(rays.far), rays.S, _p(v), *_ptr3(go), *_ptr3(w),
                                           _p(gv), *_ptr3(gpr), _p(gpar), spec.contraction, spec.contract_a)
    assert rc == 0
    return gv, gpr, gpar


def splat_mlp_relu_slack(spec: GridSpec, rays: Rays, features, g: SplatMlp, grad_out, theta_weight,
                         band: float = 2e-5):
    """Elementwise bound of how much the g_s Splatter's gradients (features,
    prior, params) may change when a g_s ReLU decision with |z| < band * scale
    flips (lp_oracle.cpp lpo_splat_mlp_relu_slack). Returns (slack_features,
    slack_prior planes, slack_params)."""
    v = _d(features).reshape(rays.n, g.C_in)
    sv = np.zeros((rays.n, g.C_in))
    spr = [np.zeros_like(a) for a in g.prior]
    spar = np.zeros_like(g.params)
    go = [_d(a) for a in grad_out]
    w = [_d(a) for a in theta_weight]
    rc = lib().lpo_splat_mlp_relu_slack(*spec._geom(), *g._args(), 0, rays.n, _p(rays.o), _p(rays.d),
                                        _p(rays.near), _p(rays.far), rays.S, _p(v), *_ptr3(go), *_ptr3(w),
                                        float(band), _p(sv), *_ptr3(spr), _p(spar), spec.contraction,
                                        spec.contract_a)
    assert rc == 0
    return sv, spr, spar
