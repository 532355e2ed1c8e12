"""PyTorch-facing API of the fused renderer (marshalling only; the math runs in
liblp_b200.so). PyTorch provides device memory and streams.

    field = Field(kind, planes, widths, params)      # CUDA fp32 tensors
    out, tau = render(field, origins, dirs, near, far, n_samples, bg)   # autograd-aware

The autograd Function saves only the per-ray optical depth tau (one scalar per
ray) besides the inputs, so the memory of a forward+backward step is
O(1) per ray in the number of samples.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch

from . import _lib

TRIPLANE = _lib.LP_GRID_TRIPLANE
VOXEL = _lib.LP_GRID_VOXEL
CONTRACT_NONE = _lib.LP_CONTRACT_NONE
CONTRACT_PER_AXIS = _lib.LP_CONTRACT_PER_AXIS
CONTRACT_RADIAL = _lib.LP_CONTRACT_RADIAL


def _req(t: torch.Tensor, name: str, shape=None) -> torch.Tensor:
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if t.device.type != "cuda":
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path)")
    if t.dtype != torch.float32:
        raise TypeError(f"{name} must be float32")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    return t


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _same_device(device, **tensors):
    for name, t in tensors.items():
        if t is not None and t.device != device:
            raise ValueError(f"{name} is on {t.device}, expected {device} (one device per call)")


def _launch(device, fn, *args):
    """One ABI call with `device` current, enqueued on that device's current
    stream (tensors on cuda:N launch on cuda:N, not on the current device)."""
    with torch.cuda.device(device):
        _lib.check(fn(*args, ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)))


@dataclass
class Field:
    """theta (3 planes [H][W][K], [W][D][K], [D][H][K] or one volume [H][W][D][K])
    plus the packed MLP parameters (include/lp.h). `contraction` / `contract_scale`
    select the scene contraction of sample points (lp_contraction)."""
    kind: int
    planes: List[torch.Tensor]
    widths: Sequence[int]
    params: torch.Tensor
    contraction: int = CONTRACT_NONE
    contract_scale: float = 1.0
    dir_freqs: int = 0          # F > 0: view-dependent field g_sigma(h), g_v(h, direnc(d)) (include/lp.h)

    def __post_init__(self):
        if self.kind == TRIPLANE:
            if len(self.planes) != 3:
                raise ValueError("triplane needs 3 planes")
            H, W, K = self.planes[0].shape
            D = self.planes[1].shape[1]
            exp = [(H, W, K), (W, D, K), (D, H, K)]
        elif self.kind == VOXEL:
            if len(self.planes) != 1:
                raise ValueError("voxel grid needs 1 volume")
            H, W, D, K = self.planes[0].shape
            exp = [(H, W, D, K)]
        else:
            raise ValueError(f"bad kind {self.kind}")
        for i, (p, s) in enumerate(zip(self.planes, exp)):
            _req(p, f"planes[{i}]", s)
        self.H, self.W, self.D, self.K = int(H), int(W), int(D), int(K)
        self.widths = tuple(int(w) for w in self.widths)
        _req(self.params, "params")
        cnt = lambda w: sum(w[i + 1] * w[i] + w[i + 1] for i in range(len(w) - 1))
        if self.dir_freqs:
            w = list(self.widths)
            n = cnt(w[:-1] + [1]) + cnt([w[0] + 6 * self.dir_freqs] + w[1:-1] + [w[-1] - 1])
        else:
            n = cnt(self.widths)
        if self.params.numel() != n:
            raise ValueError(f"params has {self.params.numel()} elements, widths {self.widths} need {n}")
        self.C = self.widths[-1] - 1

    def c_grid(self, planes=None) -> _lib.LpGrid:
        planes = self.planes if planes is None else planes
        return _lib.make_grid(self.kind, self.H, self.W, self.D, self.K, [p.data_ptr() for p in planes],
                              self.contraction, self.contract_scale)

    def c_mlp(self, params=None) -> _lib.LpMlp:
        params = self.params if params is None else params
        return _lib.make_mlp(self.widths, params.data_ptr(), self.dir_freqs)


def _c_rays(origins, dirs, near, far, n_samples) -> _lib.LpRays:
    M = origins.shape[0]
    _req(origins, "origins", (M, 3))
    _req(dirs, "dirs", (M, 3))
    _req(near, "near", (M,))
    _req(far, "far", (M,))
    return _lib.make_rays(M, origins.data_ptr(), dirs.data_ptr(), near.data_ptr(), far.data_ptr(), int(n_samples))


def render_forward(field: Field, origins, dirs, near, far, n_samples: int, bg=None, out=None, tau=None,
                   depth=None, return_depth: bool = False):
    """Eq. 1 forward. Returns (out [M][C], tau [M]), plus depth [M] (expected
    depth sum_j w_j t_j) when return_depth or a `depth` buffer is given."""
    M = origins.shape[0]
    rays = _c_rays(origins, dirs, near, far, n_samples)
    if bg is not None:
        _req(bg, "bg", (field.C,))
    out = torch.empty((M, field.C), device=origins.device, dtype=torch.float32) if out is None else out
    tau = torch.empty((M,), device=origins.device, dtype=torch.float32) if tau is None else tau
    _req(out, "out", (M, field.C))
    _req(tau, "tau", (M,))
    if return_depth and depth is None:
        depth = torch.empty((M,), device=origins.device, dtype=torch.float32)
    if depth is not None:
        _req(depth, "depth", (M,))
    _same_device(origins.device, dirs=dirs, near=near, far=far, bg=bg, out=out, tau=tau, depth=depth,
                 params=field.params, **{f"planes{i}": p for i, p in enumerate(field.planes)})
    g, m = field.c_grid(), field.c_mlp()
    _launch(origins.device, _lib.lib.lp_render_forward, ctypes.byref(g), ctypes.byref(m), ctypes.byref(rays), _ptr(bg),
            _ptr(out), _ptr(tau), _ptr(depth))
    return (out, tau) if depth is None else (out, tau, depth)


def render_backward(field: Field, origins, dirs, near, far, n_samples: int, tau, grad_out, grad_tau=None,
                    bg=None, grad_planes=None, grad_params=None, grad_depth=None):
    """Eq. 3 backward. Accumulates into (and returns) grad_planes, grad_params."""
    M = origins.shape[0]
    rays = _c_rays(origins, dirs, near, far, n_samples)
    _req(tau, "tau", (M,))
    _req(grad_out, "grad_out", (M, field.C))
    if grad_tau is not None:
        _req(grad_tau, "grad_tau", (M,))
    if grad_depth is not None:
        _req(grad_depth, "grad_depth", (M,))
    if bg is not None:
        _req(bg, "bg", (field.C,))
    if grad_planes is None:
        grad_planes = [torch.zeros_like(p) for p in field.planes]
    if grad_params is None:
        grad_params = torch.zeros_like(field.params)
    for i, (gp, p) in enumerate(zip(grad_planes, field.planes)):
        _req(gp, f"grad_planes[{i}]", p.shape)
    _req(grad_params, "grad_params", field.params.shape)
    _same_device(origins.device, dirs=dirs, near=near, far=far, bg=bg, tau=tau, grad_out=grad_out,
                 grad_tau=grad_tau, grad_depth=grad_depth, params=field.params, grad_params=grad_params,
                 **{f"planes{i}": p for i, p in enumerate(field.planes)},
                 **{f"grad_planes{i}": p for i, p in enumerate(grad_planes)})
    g, m = field.c_grid(), field.c_mlp()
    gptr = _lib.ptr_array3([t.data_ptr() for t in grad_planes])
    _launch(origins.device, _lib.lib.lp_render_backward, ctypes.byref(g), ctypes.byref(m), ctypes.byref(rays), _ptr(bg),
            _ptr(tau), _ptr(grad_out), _ptr(grad_tau), _ptr(grad_depth), gptr,
            _ptr(grad_params))
    return grad_planes, grad_params


class _RenderFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, geom, n_samples, origins, dirs, near, far, bg, params, *planes):
        kind, widths, contraction, cscale, dfreq = geom
        field = Field(kind, list(planes), widths, params, contraction, cscale, dfreq)
        out, tau, depth = render_forward(field, origins, dirs, near, far, n_samples, bg, return_depth=True)
        ctx.save_for_backward(origins, dirs, near, far, bg if bg is not None else torch.empty(0), params, tau,
                              *planes)
        ctx.meta = (geom, n_samples, bg is not None)
        return out, tau, depth

    @staticmethod
    def backward(ctx, grad_out, grad_tau, grad_depth):
        (kind, widths, contraction, cscale, dfreq), n_samples, has_bg = ctx.meta
        origins, dirs, near, far, bg, params, tau, *planes = ctx.saved_tensors
        field = Field(kind, list(planes), widths, params, contraction, cscale, dfreq)
        go = grad_out.contiguous() if grad_out is not None else torch.zeros((origins.shape[0], field.C),
                                                                           device=origins.device)
        gt = grad_tau.contiguous() if grad_tau is not None else None
        gd = grad_depth.contiguous() if grad_depth is not None else None
        gplanes, gparams = render_backward(field, origins, dirs, near, far, n_samples, tau, go, gt,
                                           bg if has_bg else None, grad_depth=gd)
        return (None, None, None, None, None, None, None, gparams, *gplanes)


def render(field: Field, origins, dirs, near, far, n_samples: int, bg=None, return_depth: bool = False):
    """Differentiable fused render: returns (out [M][C], tau [M]) -- and the
    expected depth [M] with return_depth; gradients flow to field.params and
    field.planes (not to rays, near/far or bg)."""
    geom = (field.kind, tuple(field.widths), int(field.contraction), float(field.contract_scale),
            int(field.dir_freqs))
    out, tau, depth = _RenderFn.apply(geom, int(n_samples), origins, dirs, near, far, bg, field.params,
                                      *field.planes)
    return (out, tau, depth) if return_depth else (out, tau)


def fwd_bwd_host(field: Field, origins_h, dirs_h, near_h, far_h, n_samples: int, grad_out_h, grad_tau_h=None,
                 bg_h=None, out_h=None, tau_h=None, grad_planes=None, grad_params=None, workspace=None):
    """End-to-end step through lp_render_fwd_bwd_host: host (pinned) inputs,
    host outputs, device-resident field and gradients. Synchronises."""
    M = origins_h.shape[0]
    C = field.C
    for name, t, shape in (("origins", origins_h, (M, 3)), ("dirs", dirs_h, (M, 3)), ("near", near_h, (M,)),
                           ("far", far_h, (M,)), ("grad_out", grad_out_h, (M, C)), ("grad_tau", grad_tau_h, (M,)),
                           ("bg", bg_h, (C,)), ("out", out_h, (M, C)), ("tau", tau_h, (M,))):
        if t is None and name in ("grad_tau", "bg", "out", "tau"):
            continue
        if not isinstance(t, torch.Tensor) or t.device.type != "cpu" or t.dtype != torch.float32 \
                or not t.is_contiguous() or tuple(t.shape) != shape:
            raise ValueError(f"{name} must be a contiguous float32 host tensor of shape {shape}")
    rays = _lib.make_rays(M, origins_h.data_ptr(), dirs_h.data_ptr(), near_h.data_ptr(), far_h.data_ptr(),
                          int(n_samples))
    if out_h is None:
        out_h = torch.empty((M, field.C), dtype=torch.float32, pin_memory=True)
    if tau_h is None:
        tau_h = torch.empty((M,), dtype=torch.float32, pin_memory=True)
    need = _lib.lib.lp_fwd_bwd_host_workspace_bytes(M, field.C)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=field.params.device)
    if grad_planes is None:
        grad_planes = [torch.zeros_like(p) for p in field.planes]
    if grad_params is None:
        grad_params = torch.zeros_like(field.params)
    g, m = field.c_grid(), field.c_mlp()
    gptr = _lib.ptr_array3([t.data_ptr() for t in grad_planes])
    _launch(field.params.device, _lib.lib.lp_render_fwd_bwd_host,
            ctypes.byref(g), ctypes.byref(m), ctypes.byref(rays), _ptr(bg_h), _ptr(grad_out_h), _ptr(grad_tau_h),
            _ptr(out_h), _ptr(tau_h), gptr, _ptr(grad_params), ctypes.c_void_p(workspace.data_ptr()),
            ctypes.c_size_t(workspace.numel()))
    return out_h, tau_h, grad_planes, grad_params, workspace


def set_l2_persist(hit_ratio: float):
    _lib.check(_lib.lib.lp_set_l2_persist(float(hit_ratio)))
