import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import workload as wl, oracle
from tests.gpu_problem import problem_np, to_cuda, oracle_field, oracle_rays, unambiguous
from tests.helpers import rel_inf
import paper_2404_19760_b200 as lpb

pb = unambiguous(problem_np("c2", n=256, sigma_bias=-30.0))
field, t = to_cuda(pb)
S = pb["cfg"].S
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
    a = gpl[0].cpu().numpy(); b = gg[0]
    if np.abs(b).max() == 0:
        errs.append((np.abs(a).max(), i, 0, 0)); continue
    e = np.abs(a-b); j = np.unravel_index(np.argmax(e), e.shape)
    errs.append((rel_inf(a, b), i, j, (a[j], b[j], np.abs(b).max())))
errs.sort(key=lambda x: -x[0])
for e in errs[:6]:
    print(e)
    i = e[1]
    print("   o", pb["o"][i], "d", pb["d"][i], "near", pb["near"][i], "far", pb["far"][i])
print("median", np.median([e[0] for e in errs]))
