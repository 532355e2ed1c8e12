"""PyTorch-facing API of the Splatter (include/lp.h lp_splat_*; marshalling only).

    grid = SplatGrid(VOXEL, (160, 160, 160), K=32)
    planes = splat(grid, origins, dirs, near, far, n_samples, features)   # autograd-aware

Pixel rays expand into the renderer's R+1 equispaced points, each inheriting
the pixel's feature; features are pushed into theta with the sampling
weights of h and the scalar 1 into theta_weight; the result is
theta / theta_weight. The backward w.r.t. the features mirrors the
renderer's gather with theta_weight cached.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Optional, Tuple

import torch

from . import _lib
from .render import CONTRACT_NONE, TRIPLANE, VOXEL, _c_rays, _ptr, _launch, _req


@dataclass
class SplatGrid:
    """Shape of the splat target: kind, (H, W, D), K channels, contraction."""
    kind: int
    dims: Tuple[int, int, int]
    K: int
    contraction: int = CONTRACT_NONE
    contract_scale: float = 1.0

    def shapes(self, K: Optional[int] = None) -> List[tuple]:
        K = self.K if K is None else K
        H, W, D = self.dims
        if self.kind == TRIPLANE:
            return [(H, W, K), (W, D, K), (D, H, K)]
        if self.kind == VOXEL:
            return [(H, W, D, K)]
        raise ValueError(f"bad kind {self.kind}")

    def c_grid(self) -> _lib.LpGrid:
        H, W, D = self.dims
        return _lib.make_grid(self.kind, H, W, D, self.K, [], self.contraction, self.contract_scale)

    def zeros(self, device, K: Optional[int] = None) -> List[torch.Tensor]:
        return [torch.zeros(s, device=device, dtype=torch.float32) for s in self.shapes(K)]


def _planes(grid: SplatGrid, ts, name, K=None):
    shapes = grid.shapes(K)
    if len(ts) != len(shapes):
        raise ValueError(f"{name}: expected {len(shapes)} tensors")
    for i, (t, s) in enumerate(zip(ts, shapes)):
        _req(t, f"{name}[{i}]", s)
    return _lib.ptr_array3([t.data_ptr() for t in ts])


def splat_forward(grid: SplatGrid, origins, dirs, near, far, n_samples: int, features, theta=None, weight=None):
    """Accumulate the unnormalised splat: returns (theta planes, theta_weight planes)."""
    M = origins.shape[0]
    rays = _c_rays(origins, dirs, near, far, n_samples)
    _req(features, "features", (M, grid.K))
    theta = grid.zeros(origins.device) if theta is None else theta
    weight = grid.zeros(origins.device, 1) if weight is None else weight
    g = grid.c_grid()
    _launch(origins.device, _lib.lib.lp_splat_forward, ctypes.byref(g), ctypes.byref(rays), _ptr(features),
            _planes(grid, theta, "theta"), _planes(grid, weight, "weight", 1))
    return theta, weight


def splat_normalize(grid: SplatGrid, theta, weight, out=None):
    """theta / theta_weight per cell (0 where no weight landed)."""
    out = [torch.empty_like(t) for t in theta] if out is None else out
    g = grid.c_grid()
    _launch(theta[0].device, _lib.lib.lp_splat_normalize, ctypes.byref(g), _planes(grid, theta, "theta"),
            _planes(grid, weight, "weight", 1), _planes(grid, out, "out"))
    return out


def splat_backward(grid: SplatGrid, origins, dirs, near, far, n_samples: int, grad_out, weight,
                   grad_features=None):
    """dL/d(features) of the normalised splat, theta_weight cached from the forward."""
    M = origins.shape[0]
    rays = _c_rays(origins, dirs, near, far, n_samples)
    gf = torch.empty((M, grid.K), device=origins.device, dtype=torch.float32) if grad_features is None \
        else grad_features
    _req(gf, "grad_features", (M, grid.K))
    g = grid.c_grid()
    _launch(origins.device, _lib.lib.lp_splat_backward, ctypes.byref(g), ctypes.byref(rays), _planes(grid, grad_out, "grad_out"),
            _planes(grid, weight, "weight", 1), _ptr(gf))
    return gf


class _SplatFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, geom, n_samples, origins, dirs, near, far, features):
        grid = SplatGrid(*geom)
        theta, weight = splat_forward(grid, origins, dirs, near, far, n_samples, features)
        out = splat_normalize(grid, theta, weight, out=theta)   # in place: theta itself is not kept
        ctx.save_for_backward(origins, dirs, near, far, *weight)
        ctx.meta = (geom, n_samples)
        return tuple(out)

    @staticmethod
    def backward(ctx, *grad_out):
        geom, n_samples = ctx.meta
        origins, dirs, near, far, *weight = ctx.saved_tensors
        grid = SplatGrid(*geom)
        go = [g.contiguous() if g is not None else torch.zeros(s, device=origins.device)
              for g, s in zip(grad_out, grid.shapes())]
        gf = splat_backward(grid, origins, dirs, near, far, n_samples, go, weight)
        return (None, None, None, None, None, None, gf)


def splat(grid: SplatGrid, origins, dirs, near, far, n_samples: int, features) -> List[torch.Tensor]:
    """Differentiable Splatter: returns the normalised planes (theta / theta_weight);
    gradients flow to `features` (the saved state is theta_weight only)."""
    geom = (grid.kind, tuple(grid.dims), grid.K, grid.contraction, grid.contract_scale)
    return list(_SplatFn.apply(geom, int(n_samples), origins, dirs, near, far, features))


# ---------------------------------------------------------------- Splatter with g_s (Eq. 2)
@dataclass
class SplatMlp:
    """g_s of Eq. 2: params packed layer by layer (W0 [hidden][C_in + K_prior + 6F], b0,
    (W1 [hidden][hidden], b1 when n_hidden = 2: the paper's 3-layer g_s), W_out [K][hidden],
    b_out), the prior grid theta^ (same kind / dims as the target, K_prior channels), C_in, dir_freqs."""
    params: torch.Tensor
    prior: List[torch.Tensor]
    C_in: int = 32
    dir_freqs: int = 4
    hidden: int = 64
    n_hidden: int = 1

    def c_struct(self, grid: "SplatGrid", params=None, prior=None) -> _lib.LpSplatMlp:
        params = self.params if params is None else params
        prior = self.prior if prior is None else prior
        Kp = int(prior[0].shape[-1])
        _planes(grid, prior, "prior", Kp)
        _req(params, "g_s params")
        m = _lib.LpSplatMlp()
        m.params, m.hidden, m.C_in, m.dir_freqs, m.K_prior = params.data_ptr(), self.hidden, self.C_in, \
            self.dir_freqs, Kp
        m.n_hidden = self.n_hidden
        for i in range(3):
            m.prior[i] = prior[i].data_ptr() if i < len(prior) else None
        return m


def splat_forward_mlp(grid: SplatGrid, origins, dirs, near, far, n_samples: int, features, gs: SplatMlp,
                      theta=None, weight=None):
    """Accumulate the g_s splat: returns (theta planes, theta_weight planes)."""
    M = origins.shape[0]
    rays = _c_rays(origins, dirs, near, far, n_samples)
    _req(features, "features", (M, gs.C_in))
    theta = grid.zeros(origins.device) if theta is None else theta
    weight = grid.zeros(origins.device, 1) if weight is None else weight
    g, m = grid.c_grid(), gs.c_struct(grid)
    _launch(origins.device, _lib.lib.lp_splat_forward_mlp, ctypes.byref(g), ctypes.byref(rays), _ptr(features), ctypes.byref(m),
            _planes(grid, theta, "theta"), _planes(grid, weight, "weight", 1))
    return theta, weight


def splat_backward_mlp(grid: SplatGrid, origins, dirs, near, far, n_samples: int, features, gs: SplatMlp,
                       grad_out, weight, grad_features=None, grad_prior=None, grad_params=None):
    """Gradients of the normalised g_s splat: (features [M][C_in] overwritten, prior
    planes and g_s params accumulated)."""
    M = origins.shape[0]
    rays = _c_rays(origins, dirs, near, far, n_samples)
    _req(features, "features", (M, gs.C_in))
    gf = torch.empty((M, gs.C_in), device=origins.device) if grad_features is None else grad_features
    gpr = [torch.zeros_like(p) for p in gs.prior] if grad_prior is None else grad_prior
    gpa = torch.zeros_like(gs.params) if grad_params is None else grad_params
    Kp = int(gs.prior[0].shape[-1])
    g, m = grid.c_grid(), gs.c_struct(grid)
    _launch(origins.device, _lib.lib.lp_splat_backward_mlp, ctypes.byref(g), ctypes.byref(rays), _ptr(features), ctypes.byref(m),
            _planes(grid, grad_out, "grad_out"), _planes(grid, weight, "weight", 1),
            _ptr(gf), _planes(grid, gpr, "grad_prior", Kp), _ptr(gpa))
    return gf, gpr, gpa


class _SplatMlpFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, geom, gsmeta, n_samples, origins, dirs, near, far, features, params, *prior):
        grid = SplatGrid(*geom)
        gs = SplatMlp(params, list(prior), *gsmeta)
        theta, weight = splat_forward_mlp(grid, origins, dirs, near, far, n_samples, features, gs)
        out = splat_normalize(grid, theta, weight, out=theta)
        ctx.save_for_backward(origins, dirs, near, far, features, params, *prior, *weight)
        ctx.meta = (geom, gsmeta, n_samples, len(prior))
        return tuple(out)

    @staticmethod
    def backward(ctx, *grad_out):
        geom, gsmeta, n_samples, npl = ctx.meta
        origins, dirs, near, far, features, params, *rest = ctx.saved_tensors
        prior, weight = rest[:npl], rest[npl:]
        grid = SplatGrid(*geom)
        gs = SplatMlp(params, list(prior), *gsmeta)
        go = [g.contiguous() if g is not None else torch.zeros(s, device=origins.device)
              for g, s in zip(grad_out, grid.shapes())]
        gf, gpr, gpa = splat_backward_mlp(grid, origins, dirs, near, far, n_samples, features, gs, go, weight)
        return (None, None, None, None, None, None, None, gf, gpa, *gpr)


def splat_mlp(grid: SplatGrid, origins, dirs, near, far, n_samples: int, features, gs: SplatMlp) -> List[torch.Tensor]:
    """Differentiable Splatter with g_s: normalised planes; gradients flow to the
    features, the prior grid and the g_s parameters."""
    geom = (grid.kind, tuple(grid.dims), grid.K, grid.contraction, grid.contract_scale)
    gsmeta = (gs.C_in, gs.dir_freqs, gs.hidden)
    return list(_SplatMlpFn.apply(geom, gsmeta, int(n_samples), origins, dirs, near, far, features, gs.params,
                                  *gs.prior))
