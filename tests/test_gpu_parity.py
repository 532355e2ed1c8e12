"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on the same
seeded inputs. Tolerances (BASELINE.json north_star): rendered images and tau
1e-4, gradients 1e-3, both as ||gpu - ref||_inf / ||ref||_inf per tensor
(DESIGN.md "Parity metric")."""
import numpy as np
import pytest

import oracle
import workload as wl
from tests.gpu_problem import oracle_reference, parity_errors, problem_np, to_cuda
from tests.helpers import rel_inf

pytestmark = pytest.mark.gpu

TOL_IMG = 1e-4
TOL_GRAD = 1e-3

# configs and the ray-subset size the oracle handles in seconds
CASES = [("c1", 4096), ("c2", 1024), ("c3", 512), ("c4", 2048), ("c5", 512), ("c3p", 256), ("c4p", 1024)]


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_19760_b200  # noqa: F401  (loads liblp_b200.so or fails)
    return torch


def _gpu_fwd_bwd(torch, pb, grad=True, depth=False):
    import paper_2404_19760_b200 as lpb
    field, t = to_cuda(pb)
    res = lpb.render_forward(field, t["o"], t["d"], t["near"], t["far"], pb["cfg"].S, t["bg"], return_depth=depth)
    tau = res[1]
    res = {k: v.cpu().numpy() for k, v in zip(("out", "tau", "depth"), res)}
    if grad:
        gpl, gpar = lpb.render_backward(field, t["o"], t["d"], t["near"], t["far"], pb["cfg"].S, tau, t["go"],
                                        t["gt"], t["bg"], grad_depth=t["gd"])
        res["gplanes"] = [g.cpu().numpy() for g in gpl]
        res["gparams"] = gpar.cpu().numpy()
    torch.cuda.synchronize()
    return res


def _oracle_fwd_bwd(pb, grad=True):
    return oracle_reference(pb, grad)


def _compare(g, r, grad=True):
    return parity_errors(g, r)


def _assert(errs):
    print(errs)
    assert errs["out"] < TOL_IMG and errs["tau"] < TOL_IMG, errs
    assert errs.get("depth", 0.0) < TOL_IMG, errs
    for k, v in errs.items():
        # g*: after the oracle's fp32-rounding ReLU slack (tests/gpu_problem.py RELU_BAND);
        # raw_* (no slack) and band* (diagnostic bands) are reported, not asserted
        if k.startswith("g"):
            assert v < TOL_GRAD, (k, errs)


@pytest.mark.parametrize("cfg,n", CASES)
def test_parity_subset(torch_cuda, cfg, n):
    """F1-F7 and B1-B7 on every config: forward images/tau and all gradients."""
    pb = problem_np(cfg, n=n)
    _assert(_compare(_gpu_fwd_bwd(torch_cuda, pb), _oracle_fwd_bwd(pb)))


RAW_CASES = CASES + [("c4v", 1024), ("c1v", 2048), ("cu", 256), ("cuv", 256), ("c4pv", 512)]


@pytest.mark.parametrize("cfg,n", RAW_CASES)
def test_gradient_precision(torch_cuda, cfg, n):
    """Precision guard of the contractions (DESIGN R14: 3-piece split-bf16 per-sample
    operands, 2-piece gradient operands), on every config and kernel family. Besides
    the parity metric (slack at the fp32 worst-case band RELU_BAND), two checks that a
    reduced-precision contraction fails:
      * the inf-norm error after the slack of a tighter band, 1e-6 -- the typical
        rounding of a length-64 fp32 dot product (~sqrt(64) u |W a|): fp32-class
        evaluations flip only decisions inside it (measured: every flip here lies
        below 1e-7), 16-bit operands flip decisions outside it;
      * the relative L2 error of the grid gradients < 1e-4 and of the MLP
        gradients < 5e-4 (measured <= 6e-6 and <= 1.1e-4), after the elementwise
        slack of the decisions within 1e-7 of their scale (reading R15: any fp32
        evaluation may take those either way). Without it the two-network 3-layer
        field (c4pv: 256 hidden decisions per sample) measured grid L2 2e-4 from
        decisions below 1e-7 alone -- its band-1e-7 inf-norm error is 5e-6.
    The 2-piece per-sample build (variants) fails one of these on
    every config here (band 1e-6: up to 4.3e-3; grid L2: 5e-5 .. 1.5e-3).
    The slack-free errors (raw_*, raw_l2_*) are reported."""
    pb = problem_np(cfg, n=n)
    g = _gpu_fwd_bwd(torch_cuda, pb)
    r = oracle_reference(pb, extra_bands=(1e-7, 1e-6))
    errs = _compare(g, r)
    sg7, sp7 = r["extra"][1e-7]

    def l2(a, b, sl):
        d = np.maximum(np.abs(np.asarray(a, np.float64) - b) - sl, 0.0)
        return float(np.linalg.norm(d) / max(np.linalg.norm(b), 1e-300))
    for i, (a, b, sl) in enumerate(zip(g["gplanes"], r["gplanes"], sg7)):
        errs[f"l2_gplane{i}"] = l2(a, b, sl)
        errs[f"raw_l2_gplane{i}"] = l2(a, b, 0.0)
    errs["l2_gparams"] = l2(g["gparams"], r["gparams"], sp7)
    errs["raw_l2_gparams"] = l2(g["gparams"], r["gparams"], 0.0)
    print(errs)
    _assert(errs)
    assert errs["band1e-06"] < TOL_GRAD, errs
    for k, v in errs.items():
        if k.startswith("l2_gplane"):
            assert v < 1e-4, (k, errs)
    assert errs["l2_gparams"] < 5e-4, errs


# scene contraction and the expected-depth
# output with its upstream gradient, on every kernel family: "cu" (the paper's
# unbounded renderer setting, 3-layer MLP -> K1tc2/K2tc2), c1 / c4 (one hidden
# layer -> K1tc/K2tc, triplane) and c2 (voxel).
NEXT_CASES = [("cu", 256, {}), ("c1", 1024, dict(contraction=2, contract_a=1.5, near_far=(0.05, 9.0))),
              ("c2", 256, dict(contraction=1, contract_a=0.7)), ("c4", 512, {}), ("c4p", 256, {})]


@pytest.mark.parametrize("cfg,n,over", NEXT_CASES)
def test_parity_depth_and_contraction(torch_cuda, cfg, n, over):
    import dataclasses
    pb = problem_np(cfg, n=n, with_gdepth=True)
    if over:
        pb["cfg"] = dataclasses.replace(pb["cfg"], **over)
        if "near_far" in over:
            pb["near"] = np.full_like(pb["near"], over["near_far"][0])
            pb["far"] = np.full_like(pb["far"], over["near_far"][1])
    g = _gpu_fwd_bwd(torch_cuda, pb, depth=True)
    r = oracle_reference(pb, depth=True)
    assert np.max(np.abs(r["depth"])) > 0.1
    _assert(_compare(g, r))


@pytest.mark.parametrize("sigma_bias,label", [(-30.0, "empty"), (60.0, "opaque"), (2.5, "dense")])
def test_parity_density_regimes(torch_cuda, sigma_bias, label):
    """Empty field (out = bg), opaque field (tau_R ~ 100: T_R denormal/zero in
    fp32, reading R12) and a dense field, c2 shapes."""
    pb = problem_np("c2", n=512, sigma_bias=sigma_bias)
    g, r = _gpu_fwd_bwd(torch_cuda, pb), _oracle_fwd_bwd(pb)
    if label == "empty":
        assert np.max(np.abs(g["out"] - pb["bg"][None])) < 1e-6
    if label == "opaque":
        assert np.max(r["tau"]) > 80
    _assert(_compare(g, r))


def test_ragged_tail_and_misses(torch_cuda):
    """M not a multiple of the 128-ray tile, rays that miss the cube (near = far,
    Delta = 0 -> out = bg, zero gradient) and minimal S = 2."""
    cfg = "c1"
    idx = np.arange(1000, dtype=np.int64) * 3 + 7
    pb = problem_np(cfg, idx=idx)
    pb["near"][::5] = pb["far"][::5] = 0.0        # forced misses
    _assert(_compare(_gpu_fwd_bwd(torch_cuda, pb), _oracle_fwd_bwd(pb)))
    for S in (2, 3):
        pb2 = dict(pb)
        pb2["cfg"] = wl.get_config(cfg, S=S)
        _assert(_compare(_gpu_fwd_bwd(torch_cuda, pb2), _oracle_fwd_bwd(pb2)))


def test_zero_rays_is_noop(torch_cuda):
    import paper_2404_19760_b200 as lpb
    torch = torch_cuda
    pb = problem_np("c1", idx=np.arange(4))
    field, t = to_cuda(pb)
    e = torch.zeros((0, 3), device="cuda")
    z = torch.zeros((0,), device="cuda")
    out, tau = lpb.render_forward(field, e, e, z, z, 8, None)
    gpl, gpar = lpb.render_backward(field, e, e, z, z, 8, tau, out)
    torch.cuda.synchronize()
    assert out.shape == (0, 3) and float(gpar.abs().sum()) == 0.0


@pytest.mark.parametrize("cfg,nsample", [("c2", 256), ("c4", 256), ("c4p", 256), ("c4v", 256), ("cuv", 128)])
def test_full_size_sampled_forward(torch_cuda, cfg, nsample):
    """At BASELINE.json's full size, in bench.py's launch configuration: the
    forward over all M rays, checked on sampled rays the oracle computes one by one."""
    import paper_2404_19760_b200 as lpb
    torch = torch_cuda
    c = wl.get_config(cfg)
    full = problem_np(cfg, idx=np.arange(c.n_rays, dtype=np.int64), with_gtau=False)
    field, t = to_cuda(full)
    out, tau = lpb.render_forward(field, t["o"], t["d"], t["near"], t["far"], c.S, t["bg"])
    torch.cuda.synchronize()
    pick = np.unique((wl.counter_uniform(9, np.arange(nsample, dtype=np.uint64), 0, 1) * c.n_rays).astype(np.int64))
    sub = problem_np(cfg, idx=pick, with_gtau=False)
    r = _oracle_fwd_bwd(sub, grad=False)
    assert rel_inf(out[pick].cpu().numpy(), r["out"]) < TOL_IMG
    assert rel_inf(tau[pick].cpu().numpy(), r["tau"]) < TOL_IMG


def test_backward_additive_over_shards_and_linear(torch_cuda):
    """Properties that hold at any size (c4 full batch of 8.4M rays is too big for
    the oracle): backward(all) == backward(first half) + backward(second half)
    (rays are independent), and backward(2p) == 2 backward(p)."""
    import paper_2404_19760_b200 as lpb
    torch = torch_cuda
    c = wl.get_config("c4")
    M = 1 << 20
    pb = problem_np("c4", idx=np.arange(M, dtype=np.int64))
    field, t = to_cuda(pb)
    out, tau = lpb.render_forward(field, t["o"], t["d"], t["near"], t["far"], c.S, t["bg"])
    g_all = lpb.render_backward(field, t["o"], t["d"], t["near"], t["far"], c.S, tau, t["go"], t["gt"], t["bg"])
    h = M // 2 + 37
    gp = [torch.zeros_like(p) for p in field.planes]
    gq = torch.zeros_like(field.params)
    for sl in (slice(0, h), slice(h, M)):
        lpb.render_backward(field, t["o"][sl].contiguous(), t["d"][sl].contiguous(), t["near"][sl].contiguous(),
                            t["far"][sl].contiguous(), c.S, tau[sl].contiguous(), t["go"][sl].contiguous(),
                            t["gt"][sl].contiguous(), t["bg"], grad_planes=gp, grad_params=gq)
    g2 = lpb.render_backward(field, t["o"], t["d"], t["near"], t["far"], c.S, tau, 2 * t["go"], 2 * t["gt"],
                             t["bg"])
    torch.cuda.synchronize()
    # fp32 accumulation order differs between the runs (atomics, per-CTA TMEM
    # accumulators over different sample sets): the gradient tolerance applies
    for a, b, d in zip(g_all[0], gp, g2[0]):
        assert rel_inf(b.cpu().numpy(), a.cpu().numpy()) < TOL_GRAD
        assert rel_inf(d.cpu().numpy(), 2 * a.cpu().numpy()) < TOL_GRAD
    assert rel_inf(gq.cpu().numpy(), g_all[1].cpu().numpy()) < TOL_GRAD
    assert rel_inf(g2[1].cpu().numpy(), 2 * g_all[1].cpu().numpy()) < TOL_GRAD


def test_memory_is_o1_per_ray(torch_cuda):
    """the fused path stores no per-sample state: peak device memory of a
    forward+backward does not depend on S, and the library allocates nothing."""
    import paper_2404_19760_b200 as lpb
    torch = torch_cuda
    peaks = []
    for S in (32, 128, 512):
        pb = problem_np("c4", idx=np.arange(65536, dtype=np.int64))
        pb["cfg"] = wl.get_config("c4", S=S)
        field, t = to_cuda(pb)
        gpl = [torch.zeros_like(p) for p in field.planes]
        gpa = torch.zeros_like(field.params)
        out = torch.empty((65536, 3), device="cuda")
        tau = torch.empty((65536,), device="cuda")
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
        free0 = torch.cuda.mem_get_info()[0]
        lpb.render_forward(field, t["o"], t["d"], t["near"], t["far"], S, t["bg"], out=out, tau=tau)
        lpb.render_backward(field, t["o"], t["d"], t["near"], t["far"], S, tau, t["go"], t["gt"], t["bg"],
                            grad_planes=gpl, grad_params=gpa)
        torch.cuda.synchronize()
        peaks.append(torch.cuda.max_memory_allocated() - base)
        assert torch.cuda.mem_get_info()[0] == free0
        del field, t, gpl, gpa, out, tau
    assert peaks[0] == peaks[1] == peaks[2] == 0


def test_autograd_render(torch_cuda):
    """The autograd Function routes to the same kernels (c1 shapes)."""
    import paper_2404_19760_b200 as lpb
    torch = torch_cuda
    pb = problem_np("c1", n=4096)
    field, t = to_cuda(pb)
    field.params.requires_grad_(True)
    for p in field.planes:
        p.requires_grad_(True)
    out, tau = lpb.render(field, t["o"], t["d"], t["near"], t["far"], pb["cfg"].S, t["bg"])
    loss = (out * t["go"]).sum() + (tau * t["gt"]).sum()
    loss.backward()
    r = _oracle_fwd_bwd(pb)
    g = dict(out=out.detach().cpu().numpy(), tau=tau.detach().cpu().numpy(),
             gplanes=[p.grad.cpu().numpy() for p in field.planes], gparams=field.params.grad.cpu().numpy())
    _assert(_compare(g, r))


def test_autograd_render_depth_contracted(torch_cuda):
    """render(..., return_depth=True) on a contracted field: the depth output and its
    upstream gradient flow through the autograd Function."""
    import dataclasses

    import paper_2404_19760_b200 as lpb
    pb = problem_np("c1", n=2048, with_gdepth=True)
    pb["cfg"] = dataclasses.replace(pb["cfg"], contraction=1, contract_a=1.2)
    pb["far"] = pb["far"] * 3.0
    field, t = to_cuda(pb)
    field.params.requires_grad_(True)
    for p in field.planes:
        p.requires_grad_(True)
    out, tau, depth = lpb.render(field, t["o"], t["d"], t["near"], t["far"], pb["cfg"].S, t["bg"], return_depth=True)
    loss = (out * t["go"]).sum() + (tau * t["gt"]).sum() + (depth * t["gd"]).sum()
    loss.backward()
    r = oracle_reference(pb, depth=True)
    g = dict(out=out.detach().cpu().numpy(), tau=tau.detach().cpu().numpy(), depth=depth.detach().cpu().numpy(),
             gplanes=[p.grad.cpu().numpy() for p in field.planes], gparams=field.params.grad.cpu().numpy())
    _assert(_compare(g, r))


# view-dependent colour, sigma = g_sigma(h), c = g_v(h, direnc(d))
# on the K1tcv / K2tcv kernels, with depth and contraction riding along.
VD_CASES = [("c1v", 2048, {}), ("c4v", 1024, {}), ("c1v", 1024, dict(kind=wl.VOXEL)),
            ("c4v", 512, dict(contraction=1, contract_a=1.0, near_far=(0.05, 9.0))),
            # the paper's 3-layer g_sigma / g_v (K1tcv2 / K2tcv2): its renderer setting, c4's
            # scene, a voxel grid, the radial contraction, F = 5 (E = 30 direnc columns)
            ("cuv", 256, {}), ("c4pv", 512, {}), ("c4pv", 256, dict(kind=wl.VOXEL, res=40)),
            ("cuv", 256, dict(contraction=2, contract_a=1.5)), ("c4pv", 256, dict(dir_freqs=5))]


@pytest.mark.parametrize("cfg,n,over", VD_CASES)
def test_parity_view_dependent(torch_cuda, cfg, n, over):
    import dataclasses
    pb = problem_np(cfg, n=n, with_gdepth=True)
    if over:
        pb["cfg"] = dataclasses.replace(pb["cfg"], **over)
        if "kind" in over:
            pb["grid"] = wl.make_grid(pb["cfg"])
        if "dir_freqs" in over:
            pb["params"] = wl.make_params(pb["cfg"])
        if "near_far" in over:
            pb["near"] = np.full_like(pb["near"], over["near_far"][0])
            pb["far"] = np.full_like(pb["far"], over["near_far"][1])
    g = _gpu_fwd_bwd(torch_cuda, pb, depth=True)
    r = oracle_reference(pb, depth=True)
    _assert(_compare(g, r))


def test_autograd_view_dependent(torch_cuda):
    import paper_2404_19760_b200 as lpb
    pb = problem_np("c1v", n=2048)
    field, t = to_cuda(pb)
    field.params.requires_grad_(True)
    for p in field.planes:
        p.requires_grad_(True)
    out, tau = lpb.render(field, t["o"], t["d"], t["near"], t["far"], pb["cfg"].S, t["bg"])
    ((out * t["go"]).sum() + (tau * t["gt"]).sum()).backward()
    r = oracle_reference(pb)
    g = dict(out=out.detach().cpu().numpy(), tau=tau.detach().cpu().numpy(),
             gplanes=[p.grad.cpu().numpy() for p in field.planes], gparams=field.params.grad.cpu().numpy())
    _assert(_compare(g, r))


@pytest.mark.parametrize("cfg", ["c4p", "c1v", "c4pv"])
def test_ragged_tail_other_kernel_families(torch_cuda, cfg):
    """M not a multiple of the tile and minimal S on the 3-layer (K1tc2/K2tc2) and the
    view-dependent (K1tcv/K2tcv, K1tcv2/K2tcv2) kernels."""
    import dataclasses
    idx = np.arange(1000, dtype=np.int64) * 4 + 3      # within c1v's 4096 rays
    pb = problem_np(cfg, idx=idx, with_gdepth=True)
    _assert(_compare(_gpu_fwd_bwd(torch_cuda, pb, depth=True), oracle_reference(pb, depth=True)))
    pb2 = dict(pb)
    pb2["cfg"] = dataclasses.replace(pb["cfg"], S=2)
    _assert(_compare(_gpu_fwd_bwd(torch_cuda, pb2, depth=True), oracle_reference(pb2, depth=True)))


_FMA_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
from tests.gpu_problem import problem_np, oracle_reference, parity_errors, to_cuda
import paper_2404_19760_b200 as lpb
pb = problem_np({cfg!r}, n={n})
field, t = to_cuda(pb)
out, tau, depth = lpb.render_forward(field, t["o"], t["d"], t["near"], t["far"], pb["cfg"].S, t["bg"], return_depth=True)
gpl, gpar = lpb.render_backward(field, t["o"], t["d"], t["near"], t["far"], pb["cfg"].S, tau, t["go"], t["gt"], t["bg"])
g = dict(out=out.cpu().numpy(), tau=tau.cpu().numpy(), gplanes=[a.cpu().numpy() for a in gpl], gparams=gpar.cpu().numpy())
e = parity_errors(g, oracle_reference(pb))
print(e)
assert e["out"] < 1e-4 and e["tau"] < 1e-4 and all(v < 1e-3 for k, v in e.items() if k.startswith("g")), e
"""


@pytest.mark.parametrize("cfg,n", [("c1", 2048), ("c4", 1024), ("c4p", 512), ("c2", 256)])
def test_ffma_baseline_kernels_parity(torch_cuda, cfg, n):
    """The FFMA kernels K1/K2 (the A/B baseline, LP_KERNELS=fma, read once per process)
    against the oracle, in a subprocess."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LP_KERNELS="fma")
    r = subprocess.run([sys.executable, "-c", _FMA_SCRIPT.format(root=root, cfg=cfg, n=n)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
