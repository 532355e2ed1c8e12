#!/usr/bin/env python
"""Benchmark of the fused Lightplane renderer hot path (forward + backward [+ grad all-reduce]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

A step = forward (K1) + backward (K2) over this rank's rays of the config (all
SURVEY.md §8(a) rows), plus the NCCL all-reduce of the flat [grad theta | grad MLP]
buffer when N > 1 (X1). Rays are sharded contiguously over ranks (strong scaling:
the config's total ray count is fixed). Prints one JSON line on rank 0.

Metric (BASELINE.json): rays/s fwd+bwd (whole job), peak memory bytes/ray,
% roofline of the dominant kernel (K2 backward), see DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workload as wl  # noqa: E402

FALLBACK_HBM_GBS = 6650.0
FP32_LANES_PER_SM = 128
N_SM = 148
# Measured L2 reduction throughput for full 128-byte fp32 lines (scripts/red_bench.cu,
# profiles/r1_red_bench.txt): the roofline of the backward's grid-gradient scatter.
L2_RED_GBS = 6070.0
# The same per corner-vector size (K x 4 bytes: 128 B for K = 32, 64 B for K = 16, 32 B for
# K = 8), random granules of an L2-resident 24 MB buffer (scripts/red_bench.cu gran mode,
# profiles/r1_red_bench_gran.txt): the L2 reduction unit's rate is per granule, so a 64-B
# corner vector is bound by 76.5 G granules/s = 4.90 TB/s, not by the full-line payload rate.
L2_RED_GBS_BY_GRAN = {128: 6070.0, 64: 4900.0, 32: 3560.0}


# Measured line-gather ceilings of the forward's load side (scripts/red_bench.cu gather mode,
# profiles/r2/measurements_n1_n2_rayorder_redbench.txt): 8 lanes x LDG.128 per 128-B line, 4 lines
# per warp instruction, 4 in flight per lane, full occupancy. Lines drawn from a 16-line window per
# warp (every load hits L1): 164 G lines/s = 21.05 TB/s, the ceiling used for K1tc's fraction;
# random lines over a 24 MB L2-resident buffer (L1 misses served by L2): 17.67 TB/s.
GATHER_L1_GBS = 21050.0
GATHER_L2_GBS = 17670.0


def red_peak_gbs(K: int) -> float:
    return L2_RED_GBS_BY_GRAN.get(4 * K, L2_RED_GBS)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU work for the oracle baseline")
    ap.add_argument("--l2-persist", type=float, default=0.0,
                    help="hit ratio of an L2 persisting access-policy window on theta (lp_set_l2_persist; 0 = off)")
    ap.add_argument("--ray-order", default="tiled", choices=["tiled", "raster", "shuffled"],
                    help="order of the rays in the batch (workload Config.ray_order): 16x8-pixel tiles "
                         "(default), per-view raster, or a seeded shuffle of all rays of all views")
    return ap.parse_args()


def bench_config(args):
    cfg = wl.get_config(args.config)
    if args.ray_order != "tiled":
        cfg = wl.get_config(args.config, ray_order=args.ray_order)
    return cfg


# ------------------------------------------------------------------ algorithmic work
def algorithmic_red_bytes_per_sample(cfg):
    """Grid-gradient bytes the backward must reduce per sample (B6): corners x K fp32."""
    corners = 12 if cfg.kind == wl.TRIPLANE else 8
    return corners * cfg.K * 4


def algorithmic_flops_per_sample(cfg):
    """FP32 FLOPs (2 per FMA) per sample the method itself must do.
    forward  K1: interpolation corners*K + MLP
    backward K2: re-interpolation + scatter weighting 2*corners*K + MLP recompute + dX + dW = 3*MLP."""
    corners = 12 if cfg.kind == wl.TRIPLANE else 8
    w = cfg.widths
    mlp = sum(w[i] * w[i + 1] for i in range(len(w) - 1))
    if cfg.dir_freqs:   # g_sigma (K, hidden..., 1) and g_v (K + 6F, hidden..., C)
        ws, wv = list(w[:-1]) + [1], [w[0] + 6 * cfg.dir_freqs] + list(w[1:-1]) + [w[-1] - 1]
        mlp = sum(ws[i] * ws[i + 1] + wv[i] * wv[i + 1] for i in range(len(w) - 1))
    fwd = corners * cfg.K + mlp
    bwd = 2 * corners * cfg.K + 3 * mlp
    return 2 * fwd, 2 * bwd


def tensor_flops_per_sample_bwd(cfg):
    """Split-bf16 MMA FLOP the backward kernel issues per sample (6 piece products for the
    forward-type contractions, 3 for the gradient-type ones; M x N x K per tile / tile rows).
    K2tc: Z 6 x 2 K_p H, dH 3 x 2 H K_p, weight gradients 3 x 2 (2 H_p) (K_p + 16).
    K2tc2: Z1, Z2, dA1, [dW1 db1 dWo] (M 128, N H + 16), dH, [dW0 db0] (M 64, N K_p + 8).
    K2tcv2: both networks (2 x 64 units), Z1 over [h | direnc], dW1 (M 128, N 144),
    dW0 (M 128, N 80), dWo (M 128, N 16)."""
    K = cfg.K
    KP = max(K, 16)
    H = cfg.widths[1]
    HP = max(H, 64)
    if len(cfg.widths) == 4 and cfg.dir_freqs:
        return (6 * 2 * (KP * H + (KP + 32) * H) + 6 * 2 * 2 * H * H + 3 * 2 * 2 * H * H + 3 * 2 * 128 * 144
                + 3 * 2 * 2 * H * KP + 3 * 2 * 128 * 80 + 3 * 2 * 128 * 16)
    if len(cfg.widths) == 4:
        return (6 * 2 * KP * H + 6 * 2 * H * H + 3 * 2 * H * H + 3 * 2 * 128 * (H + 16) + 3 * 2 * H * KP
                + 3 * 2 * 64 * (KP + 8))
    return 6 * 2 * KP * H + 3 * 2 * H * KP + 3 * 2 * (2 * HP) * (KP + 16)


def fp32_peak_tflops(sm_mhz):
    return N_SM * FP32_LANES_PER_SM * 2 * sm_mhz * 1e6 / 1e12


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            return json.load(open(p)), "measured"
        except Exception:
            pass
    return {"hbm_gbs": FALLBACK_HBM_GBS, "sm_max_mhz": 1965.0}, "fallback"


def ncu_traffic(cfg_name, kernel="bwd"):
    """dram bytes per launch of the dominant kernel from the committed ncu capture, or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    try:
        d = json.load(open(p))
        e = d.get(cfg_name, {}).get(kernel)
        if not e:
            return None
        # captured on a reduced ray count; scale per ray to this launch
        return e
    except Exception:
        return None


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for n, v in zip(names, s[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


# What the path computes in ("Tensor-core precision"): fp32 ray I/O, fp32
# epilogues and EA state, fp32 TMEM accumulation; the tcgen05 contractions take bf16-split operands
# x = x0 + x1 (+ x2): forward-type ones (Z, Z2, g_s layers) 3 x 3 pieces / 6 products (24 significand
# bits, fp32-class), gradient-type ones (dH, dW) 2 pieces / 3 products (16 bits, ~1.5e-5 relative
# per product); sample positions and cell indices in fp64.
DTYPE_RENDER = "f32 io/accum; split-bf16 tcgen05 MMA (3-piece fwd-type, 2-piece grad-type); fp64 positions"
DTYPE_SPLAT = "f32 io/accum; split-bf16 tcgen05 MMA (g_s: 3-piece fwd-type, 2-piece grad-type)"


# ------------------------------------------------------------------ CPU oracle baseline
ORACLE_BUF_BYTES = 16e9   # host memory for the oracle's per-thread fp64 gradient copies


class OracleRate:
    """The oracle (as it stands) fwd+bwd timed on bounded ray batches of the workload.
    Per-thread gradient buffers are allocated once and accumulated into (the
    grid-sized zero + sum of a one-shot call would otherwise dominate small
    batches); the batch size adapts so each batch runs ~1/4 of the target time.
    Threads are capped so the per-thread fp64 gradient copies fit ORACLE_BUF_BYTES
    (c5's grid is 4.3 GB in fp64)."""

    def __init__(self, cfg, threads: int):
        import oracle
        from tests.gpu_problem import grid_np
        self.oracle, self.cfg = oracle, cfg
        grid = grid_np(cfg.name)
        grid_bytes = sum(g.size for g in grid) * 8
        self.threads = max(1, min(threads, int(ORACLE_BUF_BYTES // max(grid_bytes, 1))))
        self.F = oracle.Field(cfg.kind, grid, cfg.widths, wl.make_params(cfg), cfg.contraction, cfg.contract_a,
                              cfg.dir_freqs)
        self.parts = oracle.backward_buffers(self.F, self.threads)
        self.idx_all = wl.subset_indices(cfg, 1 << 17)
        self.pos = 0
        self.n = 2 * self.threads
        self.rate = None

    def batch(self, n):
        idx = np.take(self.idx_all, np.arange(self.pos, self.pos + n), mode="wrap")
        self.pos = (self.pos + n) % len(self.idx_all)
        o, d, near, far = wl.make_rays(self.cfg, idx)
        R = self.oracle.Rays(o, d, near, far, self.cfg.S)
        go = wl.make_grad_out(idx, self.cfg.C)
        t0 = time.perf_counter()
        self.oracle.render_forward_threaded(self.F, R, None, threads=self.threads)
        self.oracle.render_backward_threaded(self.F, R, go, None, None, threads=self.threads, parts=self.parts)
        return time.perf_counter() - t0

    def run(self, target_s: float):
        """Batches until >= target_s of oracle time; returns (rays/s, rays, seconds)."""
        rays, secs = 0, 0.0
        while secs < target_s:
            if self.rate is not None:
                self.n = max(self.threads, int(self.rate * max(target_s / 4, 0.25)))
            dt = self.batch(self.n)
            rays += self.n
            secs += dt
            self.rate = self.n / dt if self.rate is None else 0.5 * (self.rate + self.n / dt)
            if self.rate is None or dt < 0.05:
                self.n *= 2
        return rays / secs, rays, secs


def cpu_oracle_rate(cfg, target_s: float, threads: int):
    """N-thread oracle rate on a bounded sample (~target_s of CPU time) plus a 1-thread
    rate (~target_s / 3): (rate, rays, secs, threads used, 1-thread rate)."""
    orc = OracleRate(cfg, threads)
    orc.run(min(1.0, target_s / 8))                   # warm-up: page in, size the batch
    rate, rays, secs = orc.run(target_s)
    one = OracleRate(cfg, 1) if orc.threads > 1 else orc
    one.run(0.5)
    rate1 = one.run(max(2.0, target_s / 3))[0]
    return rate, rays, secs, orc.threads, rate1


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ reference arm (the oracle)
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = bench_config(args)
    cores = host_cores()
    per_step = max(2.0, 60.0 / max(1, args.steps + args.warmup))
    rates = []
    splat = cfg.op == "splat"
    if splat:
        cores = 1
    else:
        orc = OracleRate(cfg, cores)
        cores = orc.threads
    for i in range(args.warmup + args.steps):
        tgt = per_step if i >= args.warmup else min(per_step, 2.0)
        rate, nrays, t = cpu_splat_rate(cfg, tgt) if splat else orc.run(tgt)
        if i >= args.warmup:
            rates.append((rate, nrays, t))
    value = sum(r[1] for r in rates) / sum(r[2] for r in rates)
    ms = 1000.0 * cfg.n_rays / value / args.gpus
    line = {
        "impl": "reference", "metric": "rays/s splat fwd+bwd" if splat else "rays/s fwd+bwd", "value": value,
        "unit": "rays/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfg, args.gpus),
        "cpu_baseline": {"value": value, "unit": "rays/s", "cores": cores, "kind": "oracle",
                         "sample": f"{sum(r[1] for r in rates)} rays of {cfg.name} (x{cfg.S} samples) fwd+bwd, "
                                   f"fp64 store-all oracle, {cores} host threads, each step a bounded batch "
                                   f"of ~{per_step:.1f} s (ms_per_step extrapolates to the full {cfg.n_rays} rays)"},
        "e2e": {"value": value, "unit": "rays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(cfg, n):
    return {"workload": f"{cfg.name}: {cfg.note}", "rays": cfg.n_rays, "rays_per_gpu": cfg.n_rays // n,
            "samples_per_ray": cfg.S, "grid": ("triplane" if cfg.kind == wl.TRIPLANE else "voxel"),
            "grid_res": cfg.res, "K": cfg.K, "mlp": "->".join(map(str, cfg.widths)),
            "parallelism": f"dp{n} (rays sharded, grad all-reduce)", "ray_order": cfg.ray_order,
            "l2": "inputs larger than L2 (rays + upstream grads per step > 126 MB); theta stays L2-resident "
                  "by design (steady-state training)"}


def init_device_and_group(torch, dist, local, world):
    """One process per GPU: cuda:LOCAL_RANK and an NCCL process group. LP_DIST_BACKEND=gloo
    (with more ranks than GPUs: rank -> GPU local % count) exercises the N > 1 code path
    on a single GPU for plumbing checks only; its timings are not measurements."""
    backend = os.environ.get("LP_DIST_BACKEND", "nccl")
    dev = torch.device("cuda", local % torch.cuda.device_count() if backend != "nccl" else local)
    torch.cuda.set_device(dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    return dev


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = init_device_and_group(torch, dist, local, world)

    import paper_2404_19760_b200 as lpb
    from paper_2404_19760_b200.dist import FlatGrads, allreduce_grads, shard_range

    cfg = bench_config(args)
    if args.l2_persist > 0:
        lpb.set_l2_persist(args.l2_persist)
    M_all = cfg.n_rays
    lo, hi = shard_range(M_all, rank, world)
    M = hi - lo
    S = cfg.S

    # ---- field and flat gradient buffer [grad theta | grad MLP] (16-byte aligned pieces)
    grid = wl.make_grid(cfg)
    params = torch.from_numpy(wl.make_params(cfg)).to(dev)
    planes = [torch.from_numpy(g).to(dev) for g in grid]
    field = lpb.Field(cfg.kind, planes, cfg.widths, params, cfg.contraction, cfg.contract_a, cfg.dir_freqs)
    grads = FlatGrads([p.shape for p in planes] + [params.shape], device=dev)
    flat = grads.flat
    gplanes, gparams = grads.views[:-1], grads.views[-1]

    # ---- this rank's rays + upstream gradients, resident in HBM
    chunk = 1 << 22
    o = torch.empty((M, 3), device=dev)
    d = torch.empty((M, 3), device=dev)
    near = torch.empty((M,), device=dev)
    far = torch.empty((M,), device=dev)
    go = torch.empty((M, cfg.C), device=dev)
    for s in range(0, M, chunk):
        e = min(M, s + chunk)
        oo, dd, nn, ff = wl.make_rays(cfg, start=lo + s, count=e - s)
        o[s:e] = torch.from_numpy(oo)
        d[s:e] = torch.from_numpy(dd)
        near[s:e] = torch.from_numpy(nn)
        far[s:e] = torch.from_numpy(ff)
        go[s:e] = torch.from_numpy(wl.make_grad_out(np.arange(lo + s, lo + e), cfg.C))
    bg = None
    out = torch.empty((M, cfg.C), device=dev)
    tau = torch.empty((M,), device=dev)
    stream = torch.cuda.current_stream()

    def step(ev=None):
        flat.zero_()
        if ev:
            ev[0].record(stream)
        lpb.render_forward(field, o, d, near, far, S, bg, out=out, tau=tau)
        if ev:
            ev[1].record(stream)
        lpb.render_backward(field, o, d, near, far, S, tau, go, None, bg, grad_planes=gplanes, grad_params=gparams)
        if ev:
            ev[2].record(stream)
        allreduce_grads(grads)
        if ev:
            ev[3].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- peak memory per ray (everything allocated beyond the field and its gradients)
    torch.cuda.reset_peak_memory_stats(dev)
    step()
    torch.cuda.synchronize()
    field_bytes = sum(p.numel() * 4 for p in planes) + params.numel() * 4 + flat.numel() * 4
    peak = torch.cuda.max_memory_allocated(dev)
    bytes_per_ray = (peak - field_bytes) / M

    # ---- timed region
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        start.record(stream)
        for i in range(args.steps):
            step(evs[i])
        stop.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = start.elapsed_time(stop)
    t_fwd = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
    t_bwd = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps
    t_ar = sum(e[2].elapsed_time(e[3]) for e in evs) / args.steps
    tt = torch.tensor([total_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms_per_step = float(tt.item()) / args.steps
    value = M_all / (ms_per_step / 1000.0)

    # ---- e2e through the C-ABI host-buffer entry (pinned host inputs, host outputs)
    e2e = None
    if not args.no_e2e:
        pin = lambda t: t.cpu().pin_memory()
        oh, dh, nh, fh, goh = pin(o), pin(d), pin(near), pin(far), pin(go)
        outh = torch.empty((M, cfg.C), pin_memory=True)
        tauh = torch.empty((M,), pin_memory=True)
        ws = None
        for i in range(args.warmup + args.steps):
            if i == args.warmup:
                if world > 1:
                    dist.barrier()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
            flat.zero_()
            _, _, _, _, ws = lpb.fwd_bwd_host(field, oh, dh, nh, fh, S, goh, None, None, outh, tauh, gplanes,
                                              gparams, ws)
            if world > 1:
                allreduce_grads(grads)
                torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e_ms = float(dt.item()) * 1000.0 / args.steps
        e2e = {"value": M_all / (e2e_ms / 1000.0), "unit": "rays/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(M * (12 + 12 + 4 + 4 + 4 * cfg.C)),
               "d2h_bytes_per_step": int(M * (4 * cfg.C + 4)),
               "api": "lp_render_fwd_bwd_host (C ABI) + NCCL all-reduce when N>1"}
        del oh, dh, nh, fh, goh

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (K2tc backward, ~78% of the step). Its binding
    # resource is the L2 reduction path of the grid-gradient scatter (B6): ncu shows the
    # FP32 and tensor pipes <25% busy, HBM traffic ~70 B/ray, and the scatter's full-line
    # reds at ~half the measured line-reduction rate.
    peaks, peak_src = load_peaks()
    clk_sum = clk.summary()
    fwd_f, bwd_f = algorithmic_flops_per_sample(cfg)
    samples = M * S
    red_b = algorithmic_red_bytes_per_sample(cfg)
    achieved_red = red_b * samples / (t_bwd / 1000.0) / 1e9
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    alu_peak = fp32_peak_tflops(sm_max)
    traffic = ncu_traffic(cfg.name)
    tc_bwd_f = tensor_flops_per_sample_bwd(cfg)
    kname = (("lp_fwd_tcv2_kernel (K1tcv2)", "lp_bwd_tcv2_kernel (K2tcv2, backward)")
             if cfg.dir_freqs > 0 and len(cfg.widths) == 4 else
             ("lp_fwd_tcv_kernel (K1tcv)", "lp_bwd_tcv_kernel (K2tcv, backward)") if cfg.dir_freqs > 0 else
             ("lp_fwd_tc2_kernel (K1tc2)", "lp_bwd_tc2p_kernel (K2tc2, backward)") if len(cfg.widths) == 4 else
             ("lp_fwd_tc_kernel (K1tc)", "lp_bwd_tcp_kernel (K2tc, backward)") if cfg.K == 32 else
             ("lp_fwd_tc_kernel (K1tc)", "lp_bwd_tc_kernel (K2tc, backward)"))
    line = {
        "metric": "rays/s fwd+bwd", "value": value, "unit": "rays/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": DTYPE_RENDER, "data": "synthetic", "config": config_dict(cfg, world),
        "breakdown_ms": {"fwd": t_fwd, "bwd": t_bwd, "allreduce": t_ar},
        "peak_bytes_per_ray": bytes_per_ray,
        "roofline": {"bound": "l2_atomic", "kernel": kname[1],
                     "achieved": achieved_red, "peak": red_peak_gbs(cfg.K), "unit": "GB/s",
                     "frac": achieved_red / red_peak_gbs(cfg.K),
                     "traffic": (traffic * M / traffic_rays(cfg.name)) if traffic else None,
                     "algorithmic": f"{red_b} B of fp32 grid-gradient reductions per sample (corners x K x 4)",
                     "peak_source": f"measured: scripts/red_bench.cu red.global.add.v4.f32 of {4 * cfg.K}-B corner "
                                    "vectors into an L2-resident 24 MB buffer, profiles/r1_red_bench.txt, "
                                    "profiles/r1_red_bench_gran.txt",
                     "alu": {"achieved_tflops": bwd_f * samples / (t_bwd / 1000.0) / 1e12,
                             "peak_tflops": alu_peak,
                             "peak_source": f"FP32 FFMA {N_SM} SMs x {FP32_LANES_PER_SM} lanes x 2 x {sm_max:.0f} MHz "
                                            f"(sm_max_mhz {peak_src}); algorithmic {bwd_f} FLOP/sample"},
                     "tensor": {"issued_bf16_tflops": tc_bwd_f * samples / (t_bwd / 1000.0) / 1e12,
                                "peak_tflops": float(peaks.get("bf16_tflops", 2250.0)),
                                "peak_source": f"MEASURED_PEAKS.json bf16 ({peak_src}); issued split-bf16 "
                                               f"MMA FLOP per sample {tc_bwd_f}"},
                     "hbm": {"achieved_gbs": ((traffic * M / traffic_rays(cfg.name)) / (t_bwd / 1000.0) / 1e9)
                             if traffic else None,
                             "peak_gbs": float(peaks.get("hbm_gbs", FALLBACK_HBM_GBS)),
                             "peak_source": f"MEASURED_PEAKS.json ({peak_src}); traffic from profiles/ncu_traffic.json"},
                     "fwd_kernel": {"kernel": kname[0], "bound": "gather (L1/L2 line loads)",
                                    "achieved": red_b * samples / (t_fwd / 1000.0) / 1e9, "unit": "GB/s",
                                    "peak": GATHER_L1_GBS, "frac": red_b * samples / (t_fwd / 1000.0) / 1e9 / GATHER_L1_GBS,
                                    "frac_of_l2_random_line_gather": red_b * samples / (t_fwd / 1000.0) / 1e9 / GATHER_L2_GBS,
                                    "algorithmic": f"{red_b} B of corner vectors gathered per sample (corners x K x 4)",
                                    "peak_source": "measured: scripts/red_bench.cu gather mode, 128-B lines from a "
                                                   "16-line window per warp (L1 hits) 21.05 TB/s; random lines of a "
                                                   "24 MB buffer (L2) 17.67 TB/s"}},
        "clocks": clk_sum,
        "gpu_launches": 2 * args.steps,
    }
    if args.l2_persist > 0:
        line["config"]["l2_persist_hit_ratio"] = args.l2_persist
    if e2e:
        line["e2e"] = e2e
    if not args.no_cpu_baseline and world == 1:
        rate, nrays, t, cores, rate1 = cpu_oracle_rate(cfg, args.cpu_seconds, host_cores())
        line["cpu_baseline"] = {"value": rate, "unit": "rays/s", "cores": cores, "kind": "oracle",
                                "value_1thread": rate1,
                                "sample": f"{nrays} rays of {cfg.name} (x{cfg.S} samples) fwd+bwd, fp64 oracle, "
                                          f"{t:.1f} s on {cores} host threads (+ a 1-thread run: value_1thread)"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------ the Splatter
def cpu_splat_rate(cfg, target_s: float):
    """The oracle's Splatter fwd (+normalise) + bwd on a bounded ray sample, 1 host thread
    (its splat keeps full fp64 grids per thread)."""
    import oracle
    spec = oracle.GridSpec(cfg.kind, (cfg.res,) * 3, cfg.K, cfg.contraction, cfg.contract_a)
    gout = wl.make_grid_grad(spec.shapes())
    g = None
    if cfg.splat_mlp:
        prior = [wl.counter_uniform(9 + i, np.arange(int(np.prod(sh)), dtype=np.uint64), -1, 1).reshape(sh)
                 for i, sh in enumerate(spec.shapes())]
        g = oracle.SplatMlp(prior, cfg.widths, wl.make_mlp(cfg.widths, seed=10, hidden_bias_scale=0.2), cfg.K,
                            cfg.dir_freqs)
    idx_all = wl.subset_indices(cfg, 1 << 14)
    n, total_rays, total_t, pos = 256, 0, 0.0, 0
    while total_t < target_s:
        idx = idx_all[pos:pos + n]
        pos = (pos + n) % len(idx_all)
        R = oracle.Rays(*wl.make_rays(cfg, idx), cfg.S)
        v = wl.make_features(idx, cfg.K)
        t0 = time.perf_counter()
        if g is not None:
            out, th, wt = oracle.splat_forward_mlp(spec, R, v, g)
            oracle.splat_backward_mlp(spec, R, v, g, gout, wt)
        else:
            out, th, wt = oracle.splat_forward(spec, R, v)
            oracle.splat_backward(spec, R, gout, wt)
        total_t += time.perf_counter() - t0
        total_rays += len(idx)
    return total_rays / total_t, total_rays, total_t


def run_splat(args):
    """Splatter step: zero theta/theta_weight, splat forward (both passes), normalise,
    backward w.r.t. the features against a resident synthetic grid gradient."""
    import torch
    import torch.distributed as dist

    import paper_2404_19760_b200 as lpb
    from paper_2404_19760_b200.dist import shard_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = init_device_and_group(torch, dist, local, world)
    cfg = bench_config(args)
    lo, hi = shard_range(cfg.n_rays, rank, world)
    M, S = hi - lo, cfg.S
    grid = lpb.SplatGrid(cfg.kind, (cfg.res,) * 3, cfg.K, cfg.contraction, cfg.contract_a)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    o, d, near, far = (T(a) for a in wl.make_rays(cfg, start=lo, count=M))
    feats = T(wl.make_features(np.arange(lo, hi), cfg.K))
    gout = [T(g) for g in wl.make_grid_grad(grid.shapes())]
    gs = None
    if cfg.splat_mlp:   # g_s of Eq. 2: prior grid of the target's shape, MLP widths cfg.widths
        prior = [T(wl.counter_uniform(9 + i, np.arange(int(np.prod(sh)), dtype=np.uint64), -1, 1).reshape(sh))
                 for i, sh in enumerate(grid.shapes())]
        gs = lpb.SplatMlp(T(wl.make_mlp(cfg.widths, seed=10, hidden_bias_scale=0.2)), prior, cfg.K, cfg.dir_freqs,
                          cfg.widths[1], n_hidden=len(cfg.widths) - 2)
        gprior = [torch.zeros_like(p) for p in prior]
        gparams = torch.zeros_like(gs.params)
    theta, weight = grid.zeros(dev), grid.zeros(dev, 1)
    gf = torch.empty((M, cfg.K), device=dev)
    stream = torch.cuda.current_stream()

    def step(ev=None):
        for t in theta + weight:
            t.zero_()
        if ev:
            ev[0].record(stream)
        if gs is not None:
            lpb.splat_forward_mlp(grid, o, d, near, far, S, feats, gs, theta, weight)
        else:
            lpb.splat_forward(grid, o, d, near, far, S, feats, theta, weight)
        if world > 1:   # the splat of a sharded view batch is a sum over ranks (one all-reduce)
            for t in theta + weight:
                dist.all_reduce(t)
        if ev:
            ev[1].record(stream)
        lpb.splat_normalize(grid, theta, weight, out=theta)
        if ev:
            ev[2].record(stream)
        if gs is not None:
            lpb.splat_backward_mlp(grid, o, d, near, far, S, feats, gs, gout, weight, gf, gprior, gparams)
        else:
            lpb.splat_backward(grid, o, d, near, far, S, gout, weight, gf)
        if ev:
            ev[3].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        start.record(stream)
        for i in range(args.steps):
            step(evs[i])
        stop.record(stream)
        torch.cuda.synchronize()
    tt = torch.tensor([start.elapsed_time(stop)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = float(tt.item()) / args.steps
    t_f = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
    t_n = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps
    t_b = sum(e[2].elapsed_time(e[3]) for e in evs) / args.steps

    e2e = None
    if not args.no_e2e:   # inputs from pinned host memory every step, a checksum of the result back
        pin = lambda t: t.cpu().pin_memory()
        hs = [pin(t) for t in (o, d, near, far, feats)]
        for i in range(args.warmup + args.steps):
            if i == args.warmup:
                torch.cuda.synchronize()
                t0 = time.perf_counter()
            for dst, src in zip((o, d, near, far, feats), hs):
                dst.copy_(src, non_blocking=True)
            step()
            float(gf[0, 0].item())
        e2e_ms = (time.perf_counter() - t0) * 1000.0 / args.steps
        e2e = {"value": cfg.n_rays / (e2e_ms / 1000.0), "unit": "rays/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(M * (32 + 4 * cfg.K)), "d2h_bytes_per_step": 4,
               "api": "paper_2404_19760_b200.splat_forward / splat_normalize / splat_backward (C ABI)"}
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    corners = 12 if cfg.kind == wl.TRIPLANE else 8
    red_b = corners * (cfg.K * 4 + 4)          # feature + weight reductions per sample
    ach = red_b * M * S / (t_f / 1000.0) / 1e9
    line = {
        "metric": "rays/s splat fwd+bwd" + (" (g_s)" if gs is not None else ""), "value": cfg.n_rays / (ms / 1000.0), "unit": "rays/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": DTYPE_SPLAT if cfg.splat_mlp else "f32", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.note}", "rays": cfg.n_rays, "samples_per_ray": S,
                   "grid": "triplane" if cfg.kind == wl.TRIPLANE else "voxel", "grid_res": cfg.res, "K": cfg.K,
                   "parallelism": f"dp{world} (rays sharded, grid all-reduce)",
                   "l2": "theta + theta_weight (grid-sized, L2-resident for s2, not for s1) re-zeroed every step"},
        "breakdown_ms": {"splat_fwd": t_f, "normalize": t_n, "splat_bwd": t_b},
        "roofline": {"bound": "l2_atomic", "kernel": ("lp_splat_mlp2_fwd_kernel" if len(cfg.widths) == 4 else "lp_splat_mlp_fwd_kernel")
                     if gs is not None else "lp_splat_fwd_kernel",
                     "achieved": ach, "peak": red_peak_gbs(cfg.K),
                     "unit": "GB/s", "frac": ach / red_peak_gbs(cfg.K), "traffic": None,
                     "algorithmic": f"{red_b} B of fp32 reductions per sample (corners x (K + 1) x 4)",
                     "peak_source": "measured: scripts/red_bench.cu, profiles/r1_red_bench.txt"},
        "clocks": clk.summary(), "gpu_launches": (3 if cfg.kind == wl.TRIPLANE else 1) + 2,
    }
    line["gpu_launches"] *= args.steps
    if e2e:
        line["e2e"] = e2e
    if not args.no_cpu_baseline and world == 1:
        rate, nrays, t = cpu_splat_rate(cfg, args.cpu_seconds)
        line["cpu_baseline"] = {"value": rate, "unit": "rays/s", "cores": 1, "kind": "oracle",
                                "sample": f"{nrays} rays of {cfg.name} (x{S} points) splat fwd+bwd, fp64 oracle, "
                                          f"{t:.1f} s on 1 host thread"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def traffic_rays(cfg_name):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    return json.load(open(p))[cfg_name]["rays"]


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif wl.get_config(args.config).op == "splat":
        run_splat(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
