"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test names the part of the oracle it pins and the passage that fixes the
expected value. None of these tests re-types the oracle's own formula to get
its expectation: expectations come from closed forms, library routines
(scipy.ndimage.map_coordinates, numpy matmul), finite differences, brute force,
the paper's printed numbers (tests/golden/) or invariants.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.ndimage import map_coordinates

import oracle
import workload as wl
from tests.helpers import rel_inf, tiny_field_arrays, tiny_rays

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _field(kind, dims=(4, 5, 6), K=3, widths=(3, 5, 4), **kw):
    grid, params = tiny_field_arrays(kind, dims, K, widths, **kw)
    return oracle.Field(kind, grid, widths, params)


def _to_index(x, N):
    return (x + 1.0) * 0.5 * (N - 1)


# ---------------------------------------------------------------- O1 sampling
@pytest.mark.parametrize("kind", [wl.TRIPLANE, wl.VOXEL])
def test_sample_matches_map_coordinates(kind):
    """O1 == scipy's order-1 (multi)linear interpolation in index space
    (P:202 trilinear, P:207-210 bilinear per plane, summed), align-corners
    domain mapping (reading R8), including points on the upper boundary."""
    F = _field(kind, dims=(4, 5, 6), K=3)
    rng = wl.counter_uniform(7, np.arange(600, dtype=np.uint64), -1.0, 1.0).reshape(200, 3).astype(np.float64)
    rng[:10, 0] = 1.0      # upper boundary tie-break (reading R8)
    rng[10:20, 1] = -1.0
    rng[20:30, 2] = 1.0
    h = oracle.sample(F, rng)
    ix = _to_index(rng[:, 0], F.H)
    iy = _to_index(rng[:, 1], F.W)
    iz = _to_index(rng[:, 2], F.D)
    exp = np.zeros_like(h)
    for k in range(F.K):
        if kind == wl.VOXEL:
            exp[:, k] = map_coordinates(F.grid[0][..., k], [ix, iy, iz], order=1, mode="nearest")
        else:
            exp[:, k] = (map_coordinates(F.grid[0][..., k], [ix, iy], order=1, mode="nearest")
                         + map_coordinates(F.grid[1][..., k], [iy, iz], order=1, mode="nearest")
                         + map_coordinates(F.grid[2][..., k], [iz, ix], order=1, mode="nearest"))
    assert np.max(np.abs(h - exp)) < 1e-12


@pytest.mark.parametrize("kind", [wl.TRIPLANE, wl.VOXEL])
def test_sample_special_cases(kind):
    """vertex-coincident point returns the vertex value; voxel cell
    centre is the mean of 8 corners; constant planes c1,c2,c3 give c1+c2+c3;
    points outside [-1,1]^3 sample zero (reading R11)."""
    F = _field(kind, dims=(4, 5, 6), K=3)
    # vertex (i, j, l) = (1, 3, 2)
    x = np.array([[-1 + 2 * 1 / 3, -1 + 2 * 3 / 4, -1 + 2 * 2 / 5]])
    h = oracle.sample(F, x)[0]
    if kind == wl.VOXEL:
        exp = F.grid[0][1, 3, 2]
    else:
        exp = F.grid[0][1, 3] + F.grid[1][3, 2] + F.grid[2][2, 1]
    assert np.max(np.abs(h - exp)) < 1e-12
    # out of cube
    assert np.all(oracle.sample(F, np.array([[1.0 + 1e-9, 0, 0], [0, -1.5, 0], [0, 0, 7.0]])) == 0.0)
    if kind == wl.VOXEL:
        xc = np.array([[-1 + 2 * 1.5 / 3, -1 + 2 * 2.5 / 4, -1 + 2 * 0.5 / 5]])
        hc = oracle.sample(F, xc)[0]
        exp = F.grid[0][1:3, 2:4, 0:2].reshape(8, -1).mean(axis=0)
        assert np.max(np.abs(hc - exp)) < 1e-12
    else:
        G = oracle.Field(kind, [np.full_like(F.grid[0], 0.25), np.full_like(F.grid[1], -1.5),
                                np.full_like(F.grid[2], 4.0)], F.widths, F.params)
        pts = wl.counter_uniform(3, np.arange(90, dtype=np.uint64), -1, 1).reshape(30, 3)
        assert np.max(np.abs(oracle.sample(G, pts) - 2.75)) < 1e-12


@pytest.mark.parametrize("kind", [wl.TRIPLANE, wl.VOXEL])
def test_sample_partition_of_unity_and_affine(kind):
    """Weights are >= 0 and sum to 1: an all-ones grid samples 1 per plane.
    Piecewise multilinear: affine along an axis inside one cell."""
    F = _field(kind, dims=(5, 4, 6), K=2, widths=(2, 5, 4))
    ones = oracle.Field(kind, [np.ones_like(g) for g in F.grid], F.widths, F.params)
    pts = wl.counter_uniform(9, np.arange(300, dtype=np.uint64), -1, 1).reshape(100, 3)
    expect = 3.0 if kind == wl.TRIPLANE else 1.0
    assert np.max(np.abs(oracle.sample(ones, pts) - expect)) < 1e-12
    # three collinear points along y inside one cell
    base = np.array([0.13, -1 + 2 * 1.2 / 3, 0.31])
    step = 2 / 3 * 0.3
    xs = np.stack([base, base + [0, step * 0.5, 0], base + [0, step, 0]])
    h = oracle.sample(F, xs)
    assert np.max(np.abs(h[1] - 0.5 * (h[0] + h[2]))) < 1e-12


@pytest.mark.parametrize("kind", [wl.TRIPLANE, wl.VOXEL])
def test_splat_is_adjoint_of_sample(kind):
    """B6 scatter is the transpose of O1: <splat(X,V), theta> = <V, sample(theta,X)>."""
    F = _field(kind, dims=(6, 5, 4), K=4, widths=(4, 5, 4))
    X = wl.counter_uniform(4, np.arange(3 * 500, dtype=np.uint64), -1.05, 1.05).reshape(500, 3)
    V = wl.counter_uniform(5, np.arange(4 * 500, dtype=np.uint64), -1, 1).reshape(500, 4).astype(np.float64)
    g = oracle.splat(F, X, V)
    lhs = sum(float(np.sum(gi * ti)) for gi, ti in zip(g, F.grid))
    rhs = float(np.sum(V * oracle.sample(F, X)))
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(rhs))


# ---------------------------------------------------------------- O2 MLP
def test_mlp_special_cases_and_numpy():
    """identity single layer is the identity; zero weights give the
    bias; random 2- and 3-layer ReLU nets equal a numpy matmul chain."""
    K = 4
    eye = np.concatenate([np.eye(K).ravel(), np.zeros(K)])
    x = wl.counter_uniform(1, np.arange(40, dtype=np.uint64), -2, 2).reshape(10, K)
    assert np.max(np.abs(oracle.mlp_forward([K, K], eye, x) - x)) < 1e-15
    b = np.arange(1, K + 1, dtype=np.float64)
    zero = np.concatenate([np.zeros(K * K), b])
    assert np.max(np.abs(oracle.mlp_forward([K, K], zero, x) - b)) < 1e-15
    for widths in ([4, 7, 4], [4, 6, 5, 4]):
        p = wl.make_mlp(widths, seed=3, sigma_bias=0.1, hidden_bias_scale=0.5).astype(np.float64)
        out = oracle.mlp_forward(widths, p, x)
        a = x.astype(np.float64)
        off = 0
        for l in range(len(widths) - 1):
            fin, fout = widths[l], widths[l + 1]
            Wm = p[off:off + fin * fout].reshape(fout, fin)
            off += fin * fout
            bb = p[off:off + fout]
            off += fout
            a = a @ Wm.T + bb
            if l < len(widths) - 2:
                a = np.maximum(a, 0)
        assert np.max(np.abs(out - a)) < 1e-13


def test_mlp_vjp_fd_and_linearity():
    """MLP VJP vs central differences (fp64) and linearity in the upstream."""
    widths = [3, 6, 5, 4]
    p = wl.make_mlp(widths, seed=8, sigma_bias=0.2, hidden_bias_scale=0.3).astype(np.float64)
    x = wl.counter_uniform(2, np.arange(15, dtype=np.uint64), -1, 1).reshape(5, 3).astype(np.float64)
    u = wl.counter_uniform(6, np.arange(20, dtype=np.uint64), -1, 1).reshape(5, 4).astype(np.float64)
    gp, gx = oracle.mlp_backward(widths, p, x, u)

    def L(pp, xx):
        return float(np.sum(u * oracle.mlp_forward(widths, pp, xx)))

    eps = 1e-6
    fd_p = np.zeros_like(p)
    for i in range(len(p)):
        e = np.zeros_like(p)
        e[i] = eps
        fd_p[i] = (L(p + e, x) - L(p - e, x)) / (2 * eps)
    fd_x = np.zeros_like(x)
    for i in range(x.size):
        e = np.zeros(x.size)
        e[i] = eps
        e = e.reshape(x.shape)
        fd_x.flat[i] = (L(p, x + e) - L(p, x - e)) / (2 * eps)
    assert rel_inf(gp, fd_p) < 1e-7
    assert rel_inf(gx, fd_x) < 1e-7
    gp2, gx2 = oracle.mlp_backward(widths, p, x, 2.5 * u)
    assert rel_inf(gp2, 2.5 * gp) < 1e-14 and rel_inf(gx2, 2.5 * gx) < 1e-14


# ---------------------------------------------------------------- O4 forward closed forms
def _const_field(sigma, color, C=3, K=2):
    """All MLP weights 0: sigma = softplus(b_0), c_k = sigmoid(b_k) everywhere."""
    widths = [K, 4, 1 + C]
    grid = [wl.counter_uniform(1, np.arange(3 * 3 * 3 * K, dtype=np.uint64), -1, 1).reshape(3, 3, 3, K)]
    params = np.zeros(4 * K + 4 + (1 + C) * 4 + 1 + C)
    b = params[-(1 + C):]
    b[0] = math.log(math.expm1(sigma)) if sigma < 30 else sigma + math.log1p(-math.exp(-sigma))
    b[1:] = [math.log(c / (1 - c)) for c in color]
    return oracle.Field(wl.VOXEL, grid, widths, params)


def test_constant_density_closed_form():
    """North star: constant sigma over length L gives opacity 1 - exp(-sigma L).
    With S = R+1 samples spaced Delta (Eq. 1, reading R1):
    tau_R = S Delta sigma, out = (e^{-Delta sigma} - e^{-S Delta sigma}) c + e^{-S Delta sigma} bg."""
    sigma, col = 1.7, [0.2, 0.5, 0.9]
    F = _const_field(sigma, col)
    o, d, near, far = tiny_rays(5)
    for S in (2, 7, 64):
        rays = oracle.Rays(o, d, near, far, S)
        bg = np.array([0.3, 0.1, 0.8])
        out, tau = oracle.render_forward(F, rays, bg)
        Dl = (far.astype(np.float64) - near) / (S - 1)
        L = S * Dl
        opacity = 1 - np.exp(-sigma * L)
        assert np.max(np.abs((1 - np.exp(-tau)) - opacity)) < 1e-13
        exp = ((np.exp(-Dl * sigma) - np.exp(-L * sigma))[:, None] * np.array(col)[None]
               + np.exp(-L * sigma)[:, None] * bg[None])
        assert np.max(np.abs(out - exp)) < 1e-13


def test_spec_worked_example_golden():
    """S:252 worked example (Delta sigma = 0.1, R = 4): T_0 = e^-0.1, T_4 = e^-0.5,
    v = (e^-0.1 - e^-0.5) c; values in tests/golden/spec_s252_constant.json."""
    g = json.load(open(os.path.join(GOLDEN, "spec_s252_constant.json")))
    F = _const_field(g["sigma"], g["color"])
    o = np.array([[0.0, 0.0, -3.0]])
    d = np.array([[0.0, 0.0, 1.0]])
    rays = oracle.Rays(o, d, [g["near"]], [g["far"]], g["R"] + 1)
    out, tau = oracle.render_forward(F, rays, None)
    assert abs(math.exp(-tau[0]) - g["T_R"]) < 1e-14
    assert np.max(np.abs(out[0] - np.array(g["v"]))) < 1e-14
    _, _, T, _, _ = oracle.trace(F, o[0], d[0], g["near"], g["far"], g["R"] + 1)
    assert abs(T[0] - g["T_0"]) < 1e-14


def test_empty_field_returns_background():
    """North star: an empty field returns the background (b_sigma = -30 => sigma ~ 9.4e-14)."""
    F = _const_field(9.357622968839299e-14, [0.5, 0.5, 0.5])
    F.params[-4] = -30.0
    o, d, near, far = tiny_rays(6)
    bg = np.array([0.25, 0.6, 0.95])
    out, tau = oracle.render_forward(F, oracle.Rays(o, d, near, far, 33), bg)
    assert np.max(np.abs(out - bg[None])) < 1e-11
    assert np.max(tau) < 1e-11


def test_sample_positions():
    """F1/F2 (reading R2): x_j = o + (near + j Delta) d with
    Delta = (far - near)/R. A linear voxel field h(x) = x_0 (reproduced
    exactly by trilinear interpolation) and a single linear layer
    o_0 = h make sigma_j = softplus(x_j,0) checkable sample by sample."""
    N = 5
    lin = np.linspace(-1, 1, N)
    grid = [np.broadcast_to(lin[:, None, None, None], (N, N, N, 1)).copy()]
    widths = [1, 2]
    params = np.array([1.0, 0.0, 0.0, 0.0])   # W = [[1],[0]], b = [0, 0]
    F = oracle.Field(wl.VOXEL, grid, widths, params)
    o = np.array([-0.9, 0.1, 0.2])
    d = np.array([1.0, 0.5, -0.25])
    d /= np.linalg.norm(d)
    near, far, S = 0.1, 1.5, 9
    sig, tau, T, w, c = oracle.trace(F, o, d, near, far, S)
    Dl = (far - near) / (S - 1)
    x0 = o[0] + (near + np.arange(S) * Dl) * d[0]
    assert np.max(np.abs(sig - np.log1p(np.exp(x0)))) < 1e-14


# ---------------------------------------------------------------- O4 invariants
@pytest.mark.parametrize("kind", [wl.TRIPLANE, wl.VOXEL])
def test_transmittance_invariants(kind):
    """North star / S:281: T non-increasing; w_j >= 0; sum_{j>=1} w_j = T_0 - T_R <= 1."""
    F = _field(kind, sigma_bias=1.0)
    o, d, near, far = tiny_rays(6)
    for i in range(6):
        sig, tau, T, w, c = oracle.trace(F, o[i], d[i], near[i], far[i], 40)
        assert np.all(np.diff(T) <= 0)
        assert np.all(w >= 0) and w[0] == 0
        assert abs(w[1:].sum() - (T[0] - T[-1])) < 1e-14
        assert T[0] <= 1.0


def test_two_sample_ray_gradient_closed_form():
    """S = 2 (R = 1): out = (T_0 - T_1) c_1 + T_1 bg;
    dL/dsigma_1 = Delta T_1 (p.c_1 - p.bg), dL/dsigma_0 = -Delta (T_0 - T_1)(p.c_1) - Delta T_1 (p.bg).
    With a constant field (W = 0) dL/db_sigma = (dsigma_0 + dsigma_1) sigmoid(b_sigma) and
    dL/db_ck = w_1 p_k c_k (1 - c_k)."""
    sigma, col = 0.8, [0.3, 0.6, 0.7]
    F = _const_field(sigma, col)
    o = np.array([[0.0, 0.0, -3.0]])
    d = np.array([[0.0, 0.0, 1.0]])
    near, far = 2.5, 3.4
    rays = oracle.Rays(o, d, [near], [far], 2)
    bg = np.array([0.9, 0.2, 0.4])
    p = np.array([[0.7, -1.1, 0.35]])
    Dl = far - near
    T0, T1 = math.exp(-Dl * sigma), math.exp(-2 * Dl * sigma)
    c = np.array(col)
    out, tau = oracle.render_forward(F, rays, bg)
    assert np.max(np.abs(out[0] - ((T0 - T1) * c + T1 * bg))) < 1e-14
    gg, gp = oracle.render_backward(F, rays, p, None, bg)
    pc, pb = float(p[0] @ c), float(p[0] @ bg)
    ds1 = Dl * T1 * (pc - pb)
    ds0 = -Dl * (T0 - T1) * pc - Dl * T1 * pb
    bs = F.params[-4]
    assert abs(gp[-4] - (ds0 + ds1) / (1 + math.exp(-bs))) < 1e-14
    assert np.max(np.abs(gp[-3:] - (T0 - T1) * p[0] * c * (1 - c))) < 1e-14


# ---------------------------------------------------------------- O5 backward
def _loss(F, rays, p, gt, bg):
    out, tau = oracle.render_forward(F, rays, bg)
    return float(np.sum(p * out) + (0.0 if gt is None else np.sum(gt * tau)))


@pytest.mark.parametrize("kind,widths", [(wl.TRIPLANE, (3, 5, 4)), (wl.VOXEL, (3, 5, 4)),
                                         (wl.TRIPLANE, (3, 6, 5, 4))])
def test_backward_matches_finite_differences(kind, widths):
    """North star: analytic gradients match central finite differences on tiny
    non-cubic grids (triplane 4x5x6, voxel 3x4x5), all parameter kinds, with
    background and tau upstream terms (fp64, eps = 1e-6)."""
    dims = (4, 5, 6) if kind == wl.TRIPLANE else (3, 4, 5)
    F = _field(kind, dims=dims, K=3, widths=widths, sigma_bias=0.4)
    o, d, near, far = tiny_rays(6)
    S = 11
    rays = oracle.Rays(o, d, near, far, S)
    p = wl.counter_uniform(31, np.arange(18, dtype=np.uint64), -1, 1).reshape(6, 3).astype(np.float64)
    gt = wl.counter_uniform(32, np.arange(6, dtype=np.uint64), -1, 1).astype(np.float64)
    bg = np.array([0.2, 0.9, 0.5])
    gg, gp = oracle.render_backward(F, rays, p, gt, bg)
    eps = 1e-6
    for gi, g in enumerate(F.grid):
        fd = np.zeros_like(g)
        flat = g.reshape(-1)
        for i in range(flat.size):
            v = flat[i]
            flat[i] = v + eps
            lp = _loss(F, rays, p, gt, bg)
            flat[i] = v - eps
            lm = _loss(F, rays, p, gt, bg)
            flat[i] = v
            fd.reshape(-1)[i] = (lp - lm) / (2 * eps)
        assert np.max(np.abs(fd)) > 1e-3, "test must exercise the grid gradient"
        assert rel_inf(gg[gi], fd) < 1e-6
    fd = np.zeros_like(F.params)
    for i in range(F.params.size):
        v = F.params[i]
        F.params[i] = v + eps
        lp = _loss(F, rays, p, gt, bg)
        F.params[i] = v - eps
        lm = _loss(F, rays, p, gt, bg)
        F.params[i] = v
        fd[i] = (lp - lm) / (2 * eps)
    assert rel_inf(gp, fd) < 1e-6


@pytest.mark.parametrize("kind", [wl.TRIPLANE, wl.VOXEL])
def test_backward_eq3_equals_literal_derivative_and_is_linear(kind):
    """O5 (Eq. 3 suffix sums) == O7 (literal O(S^2) derivative of Eq. 1), and the
    backward is linear in (p, g_tau)."""
    F = _field(kind, sigma_bias=0.9)
    o, d, near, far = tiny_rays(6)
    rays = oracle.Rays(o, d, near, far, 17)
    p = wl.counter_uniform(41, np.arange(18, dtype=np.uint64), -1, 1).reshape(6, 3)
    gt = wl.counter_uniform(42, np.arange(6, dtype=np.uint64), -1, 1)
    bg = np.array([0.6, 0.3, 0.1])
    g0, p0 = oracle.render_backward(F, rays, p, gt, bg, mode=0)
    g1, p1 = oracle.render_backward(F, rays, p, gt, bg, mode=1)
    for a, b in zip(g0, g1):
        assert rel_inf(a, b) < 1e-12
    assert rel_inf(p0, p1) < 1e-12
    g2, p2 = oracle.render_backward(F, rays, -3.0 * p.astype(np.float64), -3.0 * gt.astype(np.float64), bg)
    assert rel_inf(p2, -3.0 * p0) < 1e-13
    for a, b in zip(g2, g0):
        assert rel_inf(a, -3.0 * b) < 1e-13


def test_backward_matches_torch_autograd_of_eq1():
    """Hand-derived backward == torch float64 autograd through a literal Eq. 1
    written with the T_{j-1} - T_j weights of P:244 (independent of the
    oracle's expm1 form and suffix sums); grid sampling via torch's own
    grid_sample (align_corners=True, bilinear)."""
    torch = pytest.importorskip("torch")
    F = _field(wl.TRIPLANE, dims=(4, 5, 6), K=3, widths=(3, 5, 4), sigma_bias=0.5)
    o, d, near, far = tiny_rays(6, inside_start=True)
    S = 9
    rays = oracle.Rays(o, d, near, far, S)
    p = wl.counter_uniform(51, np.arange(18, dtype=np.uint64), -1, 1).reshape(6, 3).astype(np.float64)
    bg = np.array([0.4, 0.4, 0.9])
    gg, gp = oracle.render_backward(F, rays, p, None, bg)

    planes = [torch.tensor(g, dtype=torch.float64, requires_grad=True) for g in F.grid]
    params = torch.tensor(F.params, dtype=torch.float64, requires_grad=True)
    od = torch.tensor(o, dtype=torch.float64)
    dd = torch.tensor(d, dtype=torch.float64)
    Dl = (torch.tensor(far, dtype=torch.float64) - torch.tensor(near, dtype=torch.float64)) / (S - 1)
    t = torch.tensor(near, dtype=torch.float64)[:, None] + torch.arange(S, dtype=torch.float64)[None] * Dl[:, None]
    x = od[:, None, :] + t[..., None] * dd[:, None, :]          # [M][S][3]
    assert float(x.abs().max()) <= 1.0

    def bil(plane, a, b):
        # plane [A][B][K]; grid_sample wants input [1][K][A][B], grid (x -> B axis, y -> A axis)
        inp = plane.permute(2, 0, 1)[None]
        g = torch.stack([b, a], dim=-1)[None]                  # [1][M][S][2]
        return torch.nn.functional.grid_sample(inp, g, mode="bilinear", align_corners=True)[0].permute(1, 2, 0)

    h = bil(planes[0], x[..., 0], x[..., 1]) + bil(planes[1], x[..., 1], x[..., 2]) + bil(planes[2], x[..., 2], x[..., 0])
    W0 = params[:15].reshape(5, 3)
    b0 = params[15:20]
    W1 = params[20:40].reshape(4, 5)
    b1 = params[40:44]
    z = torch.relu(h @ W0.T + b0) @ W1.T + b1
    sigma = torch.nn.functional.softplus(z[..., 0])
    col = torch.sigmoid(z[..., 1:])
    T = torch.exp(-torch.cumsum(Dl[:, None] * sigma, dim=1))   # T_j, j = 0..R
    wgt = T[:, :-1] - T[:, 1:]                                  # T_{j-1} - T_j, j = 1..R
    out = (wgt[..., None] * col[:, 1:]).sum(1) + T[:, -1:] * torch.tensor(bg)[None]
    loss = (out * torch.tensor(p)).sum()
    loss.backward()
    for a, b in zip(gg, planes):
        assert rel_inf(a, b.grad.numpy()) < 1e-10
    assert rel_inf(gp, params.grad.numpy()) < 1e-10


# ---------------------------------------------------------------- paper arithmetic
def test_paper_memory_accounting_golden():
    """P:170 (12 GB store-all MLP outputs) and P:174 (512 MB grid) are exact
    products; golden values in tests/golden/paper_accounting.json."""
    g = json.load(open(os.path.join(GOLDEN, "paper_accounting.json")))
    a = g["naive_mlp_outputs_P170"]
    assert a["M"] * a["R"] * a["L"] * a["K"] * 4 == a["bytes"] == 12 * 2 ** 30
    b = g["pull_grid_P174"]
    assert b["N"] ** 3 * b["K"] * 4 == b["bytes"] == 512 * 2 ** 20


# ---------------------------------------------------------------- parity-metric helper
@pytest.mark.parametrize("widths", [(3, 5, 4), (3, 6, 5, 4)])
def test_relu_slack_bounds_a_flipped_decision(widths):
    """The ReLU-ambiguity slack (test infrastructure for the parity metric) bounds
    the gradient jump when one hidden pre-activation crosses 0: put unit 0 of the
    first layer exactly at z = 0 on one sample, evaluate the oracle gradient with
    the bias nudged to either side (the decision flips, the forward does not
    move), and check |g+ - g-| <= slack elementwise; slack is 0 for band 0."""
    F = _field(wl.TRIPLANE, widths=widths, sigma_bias=0.4)
    o, d, near, far = tiny_rays(2, inside_start=True)
    S = 7
    rays = oracle.Rays(o[:1], d[:1], near[:1], far[:1], S)
    p = np.array([[0.7, -0.4, 0.9]])
    gt = np.array([0.3])
    bg = np.array([0.1, 0.2, 0.3])
    K, H1 = widths[0], widths[1]
    Dl = (float(far[0]) - float(near[0])) / (S - 1)
    x = o[0].astype(np.float64) + (float(near[0]) + 3 * Dl) * d[0].astype(np.float64)
    h = oracle.sample(F, x[None])[0]
    W0 = F.params[:H1 * K].reshape(H1, K)
    b0 = F.params[H1 * K:H1 * K + H1]
    F.params[H1 * K] -= float(W0[0] @ h + b0[0])       # z_0 = 0 at sample 3
    base = F.params[H1 * K]
    res = []
    for eps in (+1e-12, -1e-12):
        F.params[H1 * K] = base + eps
        res.append(oracle.render_backward(F, rays, p, gt, bg))
    F.params[H1 * K] = base
    sg, sp = oracle.relu_slack(F, rays, p, gt, bg, band=1e-9)
    z0, _ = oracle.relu_slack(F, rays, p, gt, bg, band=0.0)
    jump_p = np.abs(res[0][1] - res[1][1])
    assert jump_p.max() > 1e-6, "the flip must change the gradient"
    assert np.all(jump_p <= sp + 1e-9)
    for a, b, s in zip(res[0][0], res[1][0], sg):
        assert np.all(np.abs(a - b) <= s + 1e-9)
    assert all(np.all(z == 0) for z in z0)
