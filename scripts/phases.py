"""Per-phase warp-cycle breakdown of the tensor-core kernels (LP_PHASES variant build).
LP_LIB_PATH=paper_2404_19760_b200/variants/lib_phases.so python scripts/phases.py [config] [rays]"""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2404_19760_b200 as lpb
from paper_2404_19760_b200 import _lib
import workload as wl
cfg = wl.get_config(sys.argv[1] if len(sys.argv) > 1 else "c4")
M = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
o, d, n, f = wl.make_rays(cfg, start=0, count=M)
T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
field = lpb.Field(cfg.kind, [T(g) for g in wl.make_grid(cfg)], cfg.widths, T(wl.make_params(cfg)),
                  cfg.contraction, cfg.contract_a, cfg.dir_freqs)
o, d, n, f = T(o), T(d), T(n), T(f)
go = T(wl.make_grad_out(np.arange(M), cfg.C))
fn = _lib.lib.lp_debug_phase_cycles
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 16)()
out, tau = lpb.render_forward(field, o, d, n, f, cfg.S)
lpb.render_backward(field, o, d, n, f, cfg.S, tau, go)
torch.cuda.synchronize(); fn(buf, 1)
e0, e1, e2 = torch.cuda.Event(True), torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); out, tau = lpb.render_forward(field, o, d, n, f, cfg.S); e1.record()
lpb.render_backward(field, o, d, n, f, cfg.S, tau, go); e2.record()
torch.cuda.synchronize(); fn(buf, 0)
v = np.array(list(buf), dtype=np.float64).reshape(2, 8)
names = [["taps", "gather", "bar", "mma-issue", "mma-wait", "epilogue", "-", "-"],
         ["taps", "gather", "bar1", "mma1-wait", "epilogue", "bar2+mma2-wait", "scatter", "drained-wait"]]
if len(cfg.widths) == 4 and not cfg.dir_freqs:   # K2tc2 (lp_tc2_kernels.cuh LP_PT slots)
    # lp_bwd_tc2p_kernel: kernel-0 slots = producer (0-1) and scatter (2-3) warps (K1tc2 has no
    # timers), kernel-1 slots = compute warps
    names[0] = ["prod:empty-wait", "prod:taps+gather", "scat:staged-wait", "scat:reduce", "-", "-", "-", "-"]
    names[1] = ["-", "-", "full+Z1-wait", "epilogues", "bar+MMA2/3/4-wait", "-", "-", "-"]
if len(cfg.widths) == 3 and not cfg.dir_freqs:   # lp_bwd_tcp_kernel (K2tc, producer warps): compute slots 2-4
    names[1] = ["-", "-", "full+Z-wait", "epilogue", "MMA2-wait", "-", "-", "-"]
for k, nm in enumerate(("fwd", "bwd")):
    groups = [range(8)]
    if names[k][0].startswith("prod"):   # producer and scatter warps: shares of each role's own time
        groups = [range(2), range(2, 4)]
    parts = []
    for g in groups:
        tot = sum(v[k][i] for i in g)
        parts += [f"{names[k][i]}={v[k][i] / tot * 100:.1f}%" for i in g if v[k][i] > 0]
    print(nm, f"{(e0.elapsed_time(e1) if k == 0 else e1.elapsed_time(e2)):.2f} ms", " ".join(parts))
