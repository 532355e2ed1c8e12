"""One forward + backward of a config on a reduced ray count, for ncu captures.

    python scripts/profile_step.py --config c4 --rays 524288 [--iters 2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_19760_b200 as lpb  # noqa: E402
import workload as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--rays", type=int, default=1 << 19)
    ap.add_argument("--iters", type=int, default=2)
    a = ap.parse_args()
    cfg = wl.get_config(a.config)
    M = min(a.rays, cfg.n_rays)
    # a contiguous block of whole views from the middle of the batch
    start = (cfg.n_rays - M) // 2
    o, d, n, f = wl.make_rays(cfg, start=start, count=M)
    dev = "cuda"
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    field = lpb.Field(cfg.kind, [T(g) for g in wl.make_grid(cfg)], cfg.widths, T(wl.make_params(cfg)),
                      cfg.contraction, cfg.contract_a, cfg.dir_freqs)
    o, d, n, f = T(o), T(d), T(n), T(f)
    go = T(wl.make_grad_out(np.arange(start, start + M), cfg.C))
    gp = [torch.zeros_like(p) for p in field.planes]
    gq = torch.zeros_like(field.params)
    for _ in range(a.iters):
        out, tau = lpb.render_forward(field, o, d, n, f, cfg.S)
        lpb.render_backward(field, o, d, n, f, cfg.S, tau, go, grad_planes=gp, grad_params=gq)
    torch.cuda.synchronize()
    print("ok", a.config, M)


if __name__ == "__main__":
    main()
