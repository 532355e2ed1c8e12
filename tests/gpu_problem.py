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


def problem_np(cfg_name: str, idx=None, n: int = 2048, sigma_bias=None, with_gtau=True, zero_bg=False,
               with_gdepth=False):
    cfg = wl.get_config(cfg_name)
    if idx is None:
        idx = wl.subset_indices(cfg, n)
    idx = np.asarray(idx, dtype=np.int64)
    o, d, near, far = wl.make_rays(cfg, idx)
    return dict(
        cfg=cfg, idx=idx, grid=grid_np(cfg_name), params=wl.make_params(cfg, sigma_bias=sigma_bias),
        o=o, d=d, near=near, far=far, bg=wl.make_bg(cfg.C, zero=zero_bg), go=wl.make_grad_out(idx, cfg.C),
        gt=wl.make_grad_tau(idx) if with_gtau else None,
        gd=wl.make_grad_tau(idx, seed=6) if with_gdepth else None)


def to_cuda(pb, device="cuda"):
    import torch
    import paper_2404_19760_b200 as lpb
    cfg = pb["cfg"]
    T = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(device)
    field = lpb.Field(cfg.kind, [T(g) for g in pb["grid"]], cfg.widths, T(pb["params"]), cfg.contraction,
                      cfg.contract_a, cfg.dir_freqs)
    return field, dict(o=T(pb["o"]), d=T(pb["d"]), near=T(pb["near"]), far=T(pb["far"]), bg=T(pb["bg"]),
                       go=T(pb["go"]), gt=T(pb["gt"]), gd=T(pb.get("gd")))


def oracle_field(pb):
    import oracle
    cfg = pb["cfg"]
    return oracle.Field(cfg.kind, pb["grid"], cfg.widths, pb["params"], cfg.contraction, cfg.contract_a,
                        cfg.dir_freqs)


def oracle_rays(pb):
    import oracle
    return oracle.Rays(pb["o"], pb["d"], pb["near"], pb["far"], pb["cfg"].S)


# ReLU'(z) at a hidden pre-activation within rounding of 0 is a decision that an
# fp32 / tensor-core evaluation and the fp64 oracle may take differently (both
# are correct roundings; reading R7 sets ReLU'(0) = 0). Gradient parity allows,
# elementwise, the oracle-computed bound of what flipping such decisions can
# change (oracle.relu_slack). RELU_BAND is the
# relative |z| / (sum |W a| + |b|) below which a decision counts as ambiguous:
# ~10x the relative error of the kernels' MLP dot products.
RELU_BAND = 2e-5


def oracle_reference(pb, grad=True, threads=8, depth=False):
    """Oracle forward (+ backward and ReLU slack) on a problem; with depth, also the
    expected depth and the grad_depth term (pb["gd"])."""
    import oracle
    F, R = oracle_field(pb), oracle_rays(pb)
    res = dict(zip(("out", "tau", "depth"), oracle.render_forward_threaded(F, R, pb["bg"], threads=threads,
                                                                          return_depth=depth)))
    if grad:
        gd = pb.get("gd")
        gg, gp = oracle.render_backward_threaded(F, R, pb["go"], pb["gt"], pb["bg"], threads=threads,
                                                 grad_depth=gd)
        sg, sp = oracle.relu_slack_threaded(F, R, pb["go"], pb["gt"], pb["bg"], band=RELU_BAND, threads=threads,
                                            grad_depth=gd)
        res.update(gplanes=gg, gparams=gp, splanes=sg, sparams=sp)
    return res


def parity_errors(g, r):
    """Parity errors of a GPU result against oracle_reference()."""
    from tests.helpers import rel_inf, rel_inf_slack
    errs = dict(out=rel_inf(g["out"], r["out"]), tau=rel_inf(g["tau"], r["tau"]))
    if "depth" in g and "depth" in r:
        errs["depth"] = rel_inf(g["depth"], r["depth"])
    if "gplanes" in g and "gplanes" in r:
        for i, (a, b, s) in enumerate(zip(g["gplanes"], r["gplanes"], r["splanes"])):
            errs[f"gplane{i}"] = rel_inf_slack(a, b, s)
            errs[f"raw_gplane{i}"] = rel_inf(a, b)
        errs["gparams"] = rel_inf_slack(g["gparams"], r["gparams"], r["sparams"])
        errs["raw_gparams"] = rel_inf(g["gparams"], r["gparams"])
    return errs
