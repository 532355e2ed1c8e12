"""One small forward + backward of a kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck; scripts/sanitize.sh). Run with LP_MAX_CTAS
capped so each persistent group marches several tiles (the multi-tile and
scatter-warp hand-offs of the benchmark launch). Checks the result against the
oracle on the same rays so a run that is clean but wrong still fails.

    python scripts/sanitize_case.py CFG N S
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(cfg_name, n, S):
    import dataclasses

    import torch

    import paper_2404_19760_b200 as lpb
    import workload as wl
    from tests.gpu_problem import oracle_reference, parity_errors, problem_np, to_cuda
    if cfg_name in ("s1", "s2", "s1g", "s2g"):
        return splat(cfg_name, n, S)
    c = wl.get_config(cfg_name)
    s0 = int(c.img * c.img * 0.3) // 128 * 128
    pb = problem_np(cfg_name, idx=np.arange(s0, s0 + n, dtype=np.int64), with_gdepth=True)
    pb["cfg"] = dataclasses.replace(pb["cfg"], S=S)
    field, t = to_cuda(pb)
    out, tau, dep = lpb.render_forward(field, t["o"], t["d"], t["near"], t["far"], S, t["bg"], return_depth=True)
    gpl, gpar = lpb.render_backward(field, t["o"], t["d"], t["near"], t["far"], S, tau, t["go"], t["gt"], t["bg"],
                                    grad_depth=t["gd"])
    torch.cuda.synchronize()
    g = dict(out=out.cpu().numpy(), tau=tau.cpu().numpy(), depth=dep.cpu().numpy(),
             gplanes=[a.cpu().numpy() for a in gpl], gparams=gpar.cpu().numpy())
    e = parity_errors(g, oracle_reference(pb, depth=True))
    print(cfg_name, n, S, e)
    assert e["out"] < 1e-4 and e["tau"] < 1e-4 and e["depth"] < 1e-4, e
    assert all(v < 1e-3 for k, v in e.items() if k.startswith("g")), e


def splat(cfg_name, n, S):
    import torch

    import paper_2404_19760_b200 as lpb
    import workload as wl
    cfg = wl.get_config(cfg_name, res=40, S=S)
    idx = wl.subset_indices(cfg, n)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    o, d, nr, fr = (T(a) for a in wl.make_rays(cfg, idx))
    grid = lpb.SplatGrid(cfg.kind, (cfg.res,) * 3, 32)
    v = T(wl.make_features(idx, 32))
    gout = [T(x) for x in wl.make_grid_grad(grid.shapes())]
    if cfg.splat_mlp:
        F = 4
        widths = (32 + 32 + 6 * F, 64, 32)
        params = T(wl.make_mlp(widths, seed=120, hidden_bias_scale=0.2))
        prior = [T(wl.counter_uniform(121 + i, np.arange(int(np.prod(s)), dtype=np.uint64), -1, 1).reshape(s))
                 for i, s in enumerate(grid.shapes())]
        gs = lpb.SplatMlp(params, prior, 32, F, 64)
        th, wt = lpb.splat_forward_mlp(grid, o, d, nr, fr, S, v, gs)
        lpb.splat_normalize(grid, th, wt)
        lpb.splat_backward_mlp(grid, o, d, nr, fr, S, v, gs, gout, wt)
    else:
        th, wt = lpb.splat_forward(grid, o, d, nr, fr, S, v)
        lpb.splat_normalize(grid, th, wt)
        lpb.splat_backward(grid, o, d, nr, fr, S, gout, wt)
    torch.cuda.synchronize()
    print(cfg_name, n, S, "ok", float(wt[0].sum()))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]))
