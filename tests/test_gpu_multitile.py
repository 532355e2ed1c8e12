"""GPU parity of the multi-tile march: every group of the persistent kernels
marches several 128-ray tiles, as in bench.py's launch (c4: ~221 tiles per
group), against the fp64 oracle.

What only shows up with more than one tile per group:
the TMEM weight-gradient accumulators summed across tiles (B7 flushes once per
CTA), the scatter warps' staged/drained mbarrier phases across tile
boundaries, the per-tile reload of the ray state, and the forward's tile loop.
Two ways to get there:
  * capped grid: a subprocess with LP_MAX_CTAS=2 (read once per process,
    lp_launch.cuh) on a few thousand rays -- 4..16 tiles per group;
  * large M at the default launch (148 SMs x resident CTAs), >= 2 tiles per group.
Both assert the parity metric (inf-norm error after the fp32-rounding ReLU slack)
and report the slack-free ("raw"), tighter-band and relative-L2 errors (DESIGN.md
section 4); at 10^7..10^8 samples some hidden units always sit within fp32
rounding of 0 (measured: below 1e-6 of their scale), so those are not asserted.
Reverse march P:350-353; independent per-ray programs P:291."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from tests.gpu_problem import oracle_reference, parity_errors, problem_np, to_cuda

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL_IMG, TOL_GRAD = 1e-4, 1e-3
THREADS = max(1, min(32, os.cpu_count() or 1))


def _contiguous(cfg_name, n, start_frac=0.3):
    """n consecutive rays (whole tiles of neighbouring pixels, the layout whose
    scatter reductions collide most) starting inside view 0's image."""
    import workload as wl
    c = wl.get_config(cfg_name)
    s = int(c.img * c.img * start_frac) // 128 * 128
    return np.arange(s, s + n, dtype=np.int64) % c.n_rays


def run_case(cfg_name, n, depth=False, over=None):
    """GPU forward + backward on n contiguous rays vs the oracle; returns the error dict."""
    import dataclasses

    import torch

    import paper_2404_19760_b200 as lpb
    pb = problem_np(cfg_name, idx=_contiguous(cfg_name, n), with_gdepth=depth)
    if over:
        pb["cfg"] = dataclasses.replace(pb["cfg"], **over)
    field, t = to_cuda(pb)
    S = pb["cfg"].S
    res = lpb.render_forward(field, t["o"], t["d"], t["near"], t["far"], S, t["bg"], return_depth=depth)
    gpl, gpar = lpb.render_backward(field, t["o"], t["d"], t["near"], t["far"], S, res[1], t["go"], t["gt"],
                                    t["bg"], grad_depth=t["gd"])
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in zip(("out", "tau", "depth"), res)}
    g["gplanes"] = [a.cpu().numpy() for a in gpl]
    g["gparams"] = gpar.cpu().numpy()
    r = oracle_reference(pb, threads=THREADS, depth=depth, extra_bands=(1e-7, 1e-6))
    errs = parity_errors(g, r)
    for i, (a, b) in enumerate(zip(g["gplanes"], r["gplanes"])):
        errs[f"l2_gplane{i}"] = float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
    errs["l2_gparams"] = float(np.linalg.norm(g["gparams"] - r["gparams"]) / np.linalg.norm(r["gparams"]))
    return errs


def _assert_all(errs):
    print(errs)
    assert errs["out"] < TOL_IMG and errs["tau"] < TOL_IMG, errs
    assert errs.get("depth", 0.0) < TOL_IMG, errs
    for k, v in errs.items():
        if k.startswith("g"):   # after the fp32-rounding ReLU slack; raw_* / band* reported
            assert v < TOL_GRAD, (k, errs)



_SCRIPT = r"""
import json, sys
sys.path.insert(0, {root!r})
from tests.test_gpu_multitile import run_case
print("ERRS" + json.dumps(run_case({cfg!r}, {n}, depth={depth!r}, over={over!r})))
"""

# (config, rays, depth): kernel families K2tc (K = 8 / 16 / 32, triplane and voxel),
# K2tc2 (3-layer MLP, with contraction in cu), K2tcv (view-dependent) and K2tcv2
# (view-dependent 3-layer nets, 64-ray tiles: n / 128 tiles per CTA)
CAPPED = [("c1", 4096, False), ("c2", 2048, False), ("c4", 4096, True), ("c5", 2048, False),
          ("c4p", 2048, True), ("cu", 1024, True), ("c4v", 2048, True), ("c1v", 4096, False),
          ("cuv", 1024, True), ("c4pv", 2048, False)]


@pytest.mark.parametrize("cfg,n,depth", CAPPED)
def test_multitile_capped_grid(cfg, n, depth):
    """LP_MAX_CTAS=2: 2 persistent CTAs march all tiles (K2tc: 2 groups per CTA ->
    n / 512 tiles per group; K2tc2 / K2tcv: one group -> n / 256)."""
    pytest.importorskip("torch")
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, LP_MAX_CTAS="2")
    r = subprocess.run([sys.executable, "-c", _SCRIPT.format(root=ROOT, cfg=cfg, n=n, depth=depth, over=None)],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("ERRS")][-1]
    _assert_all(json.loads(line[4:]))


# default launch: K2tc has 148 x 2 groups, K2tc2 / K2tcv 148 x 1 -> >= 2 tiles per group
LARGE = [("c4", 81920, False), ("c4p", 40960, False), ("c4v", 40960, False), ("c4pv", 40960, False)]


@pytest.mark.parametrize("cfg,n,depth", LARGE)
def test_multitile_default_launch(cfg, n, depth):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _assert_all(run_case(cfg, n, depth=depth))


def test_fwd_bwd_host_parity():
    """lp_render_fwd_bwd_host (the e2e path: pinned host rays and upstream
    gradients in, host out/tau, device gradients) against the oracle, on more
    tiles than one wave of groups."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_19760_b200 as lpb
    pb = problem_np("c4", idx=_contiguous("c4", 81920))
    field, _ = to_cuda(pb)
    H = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    out_h, tau_h, gpl, gpar, _ = lpb.fwd_bwd_host(field, H(pb["o"]), H(pb["d"]), H(pb["near"]), H(pb["far"]),
                                                  pb["cfg"].S, H(pb["go"]), H(pb["gt"]), H(pb["bg"]))
    g = dict(out=out_h.numpy(), tau=tau_h.numpy(), gplanes=[a.cpu().numpy() for a in gpl],
             gparams=gpar.cpu().numpy())
    _assert_all(parity_errors(g, oracle_reference(pb, threads=THREADS)))
