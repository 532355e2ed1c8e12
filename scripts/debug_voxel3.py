import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import workload as wl, oracle
from tests.gpu_problem import problem_np, to_cuda, oracle_field, oracle_rays
from tests.helpers import rel_inf
import paper_2404_19760_b200 as lpb

cfg = wl.get_config("c1", kind=1)
pb = problem_np("c1", n=256)
pb["cfg"] = cfg; pb["grid"] = wl.make_grid(cfg); pb["params"] = wl.make_mlp(cfg.widths)
o, d, near, far = wl.make_rays(cfg, pb["idx"]); pb.update(o=o, d=d, near=near, far=far)
pb["go"] = np.zeros_like(pb["go"]); pb["bg"] = np.zeros(3, np.float32)
field, t = to_cuda(pb)
S = cfg.S
out, tau = lpb.render_forward(field, t["o"], t["d"], t["near"], t["far"], S, t["bg"])
F = oracle_field(pb)
M = len(pb["idx"])
errs = []
for i in range(M):
    sl = slice(i, i+1)
    f = lambda x: None if x is None else x[sl].contiguous()
    gpl, gpar = lpb.render_backward(field, f(t["o"]), f(t["d"]), f(t["near"]), f(t["far"]), S, f(tau), f(t["go"]), f(t["gt"]), t["bg"])
    torch.cuda.synchronize()
    R = oracle.Rays(pb["o"][sl], pb["d"][sl], pb["near"][sl], pb["far"][sl], S)
    gg, gp = oracle.render_backward(F, R, pb["go"][sl], pb["gt"][sl], pb["bg"])
    e = rel_inf(gpl[0].cpu().numpy(), gg[0]) if np.abs(gg[0]).max() > 0 else np.abs(gpl[0].cpu().numpy()).max()
    errs.append((e, i))
errs.sort(reverse=True)
for e, i in errs[:8]:
    print("ray", i, "err", e, "o", pb["o"][i], "d", pb["d"][i], "near", pb["near"][i], "far", pb["far"][i], "tau", tau[i].item())
    sig, tt, T, w, c = oracle.trace(F, pb["o"][i], pb["d"][i], pb["near"][i], pb["far"][i], S)
    Dl = (float(pb["far"][i]) - float(pb["near"][i]))/(S-1)
    xs = pb["o"][i].astype(np.float64)[None] + (pb["near"][i] + np.arange(S)*Dl)[:, None]*pb["d"][i].astype(np.float64)[None]
    print("   max|x|", np.abs(xs).max(axis=1)[:3], np.abs(xs).max(axis=1)[-3:])
print("median err", np.median([e for e, i in errs]))
