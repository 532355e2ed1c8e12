import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import workload as wl, oracle
from tests.gpu_problem import problem_np, to_cuda, oracle_field, oracle_rays
from tests.helpers import rel_inf
import paper_2404_19760_b200 as lpb

def run(cfgname, n, **ov):
    pb = problem_np(cfgname, n=n)
    if ov:
        cfg = wl.get_config(cfgname, **ov)
        pb = problem_np(cfgname, n=n)
        pb["cfg"] = cfg
        pb["grid"] = wl.make_grid(cfg)
        pb["params"] = wl.make_mlp(cfg.widths)
        o, d, near, far = wl.make_rays(cfg, pb["idx"])
        pb.update(o=o, d=d, near=near, far=far)
    field, t = to_cuda(pb)
    S = pb["cfg"].S
    out, tau = lpb.render_forward(field, t["o"], t["d"], t["near"], t["far"], S, t["bg"])
    gpl, gpar = lpb.render_backward(field, t["o"], t["d"], t["near"], t["far"], S, tau, t["go"], t["gt"], t["bg"])
    torch.cuda.synchronize()
    F, R = oracle_field(pb), oracle_rays(pb)
    gg, gp = oracle.render_backward_threaded(F, R, pb["go"], pb["gt"], pb["bg"], threads=8)
    for i, (a, b) in enumerate(zip(gpl, gg)):
        a = a.cpu().numpy()
        e = np.abs(a - b)
        j = np.unravel_index(np.argmax(e), e.shape)
        big = (e > 1e-3 * np.abs(b).max()).sum()
        print(cfgname, ov, "plane", i, "rel", rel_inf(a, b), "argmax", j, "gpu", a[j], "ref", b[j], "nbad", big,
              "nz_gpu", (a != 0).sum(), "nz_ref", (b != 0).sum())
    print("params rel", rel_inf(gpar.cpu().numpy(), gp))

run("c1", 512)
run("c1", 512, kind=1)              # voxel K=8
run("c2", 256, kind=0, res=64)      # triplane K=16
run("c2", 256, res=16)              # voxel 16^3 K=16
run("c2", 256)
run("c2", 64, S=32)
