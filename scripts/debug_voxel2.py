import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import workload as wl, oracle
from tests.gpu_problem import problem_np, to_cuda, oracle_field, oracle_rays
from tests.helpers import rel_inf
import paper_2404_19760_b200 as lpb

def mk(cfgname, n, **ov):
    cfg = wl.get_config(cfgname, **ov)
    pb = problem_np(cfgname, n=n)
    pb["cfg"] = cfg
    pb["grid"] = wl.make_grid(cfg)
    pb["params"] = wl.make_mlp(cfg.widths)
    o, d, near, far = wl.make_rays(cfg, pb["idx"])
    pb.update(o=o, d=d, near=near, far=far)
    return pb

def cmp(pb, label, per_ray=False):
    field, t = to_cuda(pb)
    S = pb["cfg"].S
    out, tau = lpb.render_forward(field, t["o"], t["d"], t["near"], t["far"], S, t["bg"])
    if per_ray:
        gpl = [torch.zeros_like(p) for p in field.planes]; gpar = torch.zeros_like(field.params)
        M = t["o"].shape[0]
        for i in range(M):
            sl = slice(i, i+1)
            f = lambda x: None if x is None else x[sl].contiguous()
            lpb.render_backward(field, f(t["o"]), f(t["d"]), f(t["near"]), f(t["far"]), S, f(tau), f(t["go"]), f(t["gt"]), t["bg"], grad_planes=gpl, grad_params=gpar)
    else:
        gpl, gpar = lpb.render_backward(field, t["o"], t["d"], t["near"], t["far"], S, tau, t["go"], t["gt"], t["bg"])
    torch.cuda.synchronize()
    F, R = oracle_field(pb), oracle_rays(pb)
    ro, rt = oracle.render_forward(F, R, pb["bg"])
    gg, gp = oracle.render_backward(F, R, pb["go"], pb["gt"], pb["bg"])
    print(label, "out", rel_inf(out.cpu().numpy(), ro), "tau", rel_inf(tau.cpu().numpy(), rt),
          "grid", [rel_inf(a.cpu().numpy(), b) for a, b in zip(gpl, gg)], "params", rel_inf(gpar.cpu().numpy(), gp))
    return gpl, gg

pb = mk("c1", 256, kind=1)
cmp(pb, "voxel c1 base")
cmp(pb, "voxel c1 per-ray launches", per_ray=True)
q = dict(pb); q["gt"] = None; q["bg"] = np.zeros(3, np.float32)
cmp(q, "no gtau, bg0")
q2 = dict(q); q2["go"] = np.zeros_like(pb["go"]); q2["gt"] = pb["gt"]
cmp(q2, "gtau only")
q3 = dict(q); q3["params"] = wl.make_mlp(pb["cfg"].widths, sigma_bias=-30.0)
cmp(q3, "empty field colour only")
q4 = dict(q); q4["go"] = np.ones_like(pb["go"])
cmp(q4, "p=1")
pb1 = mk("c1", 8, kind=1)
a, b = cmp(pb1, "8 rays")
a = a[0].cpu().numpy(); b = b[0]
e = np.abs(a-b); idx = np.argsort(-e.ravel())[:10]
for i in idx:
    j = np.unravel_index(i, a.shape); print(j, a[j], b[j])
