import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import workload as wl, oracle
from tests.gpu_problem import problem_np, oracle_field
cfg = wl.get_config("c1", kind=1)
pb = problem_np("c1", n=256)
pb["cfg"] = cfg; pb["grid"] = wl.make_grid(cfg); pb["params"] = wl.make_mlp(cfg.widths)
o, d, near, far = wl.make_rays(cfg, pb["idx"]); pb.update(o=o, d=d, near=near, far=far)
F = oracle_field(pb)
S = cfg.S
W0 = pb["params"][:128].reshape(16, 8).astype(np.float64)
for i in (33, 38):
    Dl = (float(far[i]) - float(near[i]))/(S-1)
    xs = o[i].astype(np.float64)[None] + (float(near[i]) + np.arange(S)*Dl)[:, None]*d[i].astype(np.float64)[None]
    h = oracle.sample(F, xs)
    z = h @ W0.T
    scale = np.abs(h) @ np.abs(W0).T
    r = np.abs(z)/scale
    j = np.unravel_index(np.argmin(r), r.shape)
    print(i, "min rel |z|", r.min(), "at", j, z[j], scale[j])
