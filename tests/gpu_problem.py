"""Seeded problems shared by the GPU parity tests, smoke() and bench.py.

Builds the same float32 inputs for both sides from `workload` (no method
arithmetic here): numpy arrays for the oracle, CUDA tensors for the library.
"""
from __future__ import annotations

import functools

import numpy as np

import workload as wl


@functools.lru_cache(maxsize=4)
def grid_np(cfg_name: str):
    return wl.make_grid(wl.get_config(cfg_name))


def problem_np(cfg_name: str, idx=None, n: int = 2048, sigma_bias=None, with_gtau=True, zero_bg=False):
    cfg = wl.get_config(cfg_name)
    if idx is None:
        idx = wl.subset_indices(cfg, n)
    idx = np.asarray(idx, dtype=np.int64)
    o, d, near, far = wl.make_rays(cfg, idx)
    return dict(
        cfg=cfg, idx=idx, grid=grid_np(cfg_name), params=wl.make_mlp(cfg.widths, sigma_bias=sigma_bias),
        o=o, d=d, near=near, far=far, bg=wl.make_bg(cfg.C, zero=zero_bg), go=wl.make_grad_out(idx, cfg.C),
        gt=wl.make_grad_tau(idx) if with_gtau else None)


def to_cuda(pb, device="cuda"):
    import torch
    import paper_2404_19760_b200 as lpb
    cfg = pb["cfg"]
    T = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(device)
    field = lpb.Field(cfg.kind, [T(g) for g in pb["grid"]], cfg.widths, T(pb["params"]))
    return field, dict(o=T(pb["o"]), d=T(pb["d"]), near=T(pb["near"]), far=T(pb["far"]), bg=T(pb["bg"]),
                       go=T(pb["go"]), gt=T(pb["gt"]))


def oracle_field(pb):
    import oracle
    cfg = pb["cfg"]
    return oracle.Field(cfg.kind, pb["grid"], cfg.widths, pb["params"])


def oracle_rays(pb):
    import oracle
    return oracle.Rays(pb["o"], pb["d"], pb["near"], pb["far"], pb["cfg"].S)


# ReLU'(z) at a hidden pre-activation within fp32 rounding of 0 is a decision that
# fp32 and fp64 may take differently (both are correct roundings; reading R7 sets
# ReLU'(0) = 0). Rays containing such a unit are compared on the forward only
# (DESIGN.md "Parity metric"). RELU_BAND is the relative |z| / (sum |W a| + |b|)
# below which the decision counts as ambiguous (~16 fp32 ulps of the MLP dot
# products; positions and cell indices are fp64 on both sides, so they add no error).
RELU_BAND = 1e-6


def unambiguous(pb, band=RELU_BAND, verbose=True):
    """Restrict a problem to the rays whose ReLU decisions are all well-conditioned."""
    import oracle
    m = oracle.min_preact(oracle_field(pb), oracle_rays(pb))
    keep = m >= band
    q = dict(pb)
    for k in ("idx", "o", "d", "near", "far", "go", "gt"):
        if q.get(k) is not None:
            q[k] = np.ascontiguousarray(q[k][keep])
    if verbose:
        print(f"relu-ambiguous rays excluded from gradient parity: {int((~keep).sum())} of {len(keep)}")
    return q
