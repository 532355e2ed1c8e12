"""Pins for the oracle's SURVEY 8(f) extensions, checked against things other than
the oracle itself:

* scene contraction CC (Supp. Eq. "contract"; reading R25):
  the a = 1 case is "the normal contract coordinates", i.e. half of the
  mip-NeRF 360 contraction x -> (2 - 1/|x|) x/|x| written out here as the
  textbook routine; the foreground maps to [-a/2, a/2]; continuity and
  limits; hand-computed values; a field that is affine in position, where
  trilinear sampling is exact, so every per-sample density has a closed form;
* expected depth (the "depths" feature of P:234; reading R26): the geometric
  series closed form under constant density, the weighted-mean bound, and the
  backward of the depth term against finite differences and the literal
  O(S^2) derivative.
"""
import math

import numpy as np
import pytest

import oracle
import workload as wl
from tests.helpers import rel_inf, tiny_field_arrays, tiny_rays


def _mipnerf360(x):
    """Barron et al. 2022 contraction: x if ||x|| <= 1 else (2 - 1/||x||) x/||x||."""
    n = np.linalg.norm(x, axis=-1, keepdims=True)
    return np.where(n <= 1.0, x, (2.0 - 1.0 / np.maximum(n, 1e-300)) * x / np.maximum(n, 1e-300))


def _pts(n=2000, scale=6.0, seed=70):
    x = wl.counter_uniform(seed, np.arange(3 * n, dtype=np.uint64), -1, 1).reshape(n, 3).astype(np.float64)
    r = wl.counter_uniform(seed + 1, np.arange(n, dtype=np.uint64), 0, 1).astype(np.float64)
    return x * (scale * r ** 2)[:, None]      # many points inside and outside the unit ball / cube


def test_contract_a1_is_half_the_mipnerf360_contraction():
    x = _pts()
    rad = oracle.contract(2, 1.0, x)
    assert np.max(np.abs(rad - 0.5 * _mipnerf360(x))) < 1e-15
    # per-axis: the same 1D map on every coordinate ("independently")
    ax = oracle.contract(1, 1.0, x)
    ref = np.stack([0.5 * _mipnerf360(x[:, k:k + 1])[:, 0] for k in range(3)], axis=1)
    assert np.max(np.abs(ax - ref)) < 1e-15


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("a", [0.25, 0.5, 1.0, 1.5, 2.0])
def test_contract_ranges_continuity_limits(mode, a):
    x = _pts()
    y = oracle.contract(mode, a, x)
    # "maps unbounded scenes into a [-1,1] cube"; strictly inside unless a = 2, where
    # (2 - a) = 0 collapses the whole background onto the cube's surface
    assert np.all(np.abs(y) < 1.0) if a < 2 else np.all(np.abs(y) <= 1.0)
    norm = np.abs(x) if mode == 1 else np.linalg.norm(x, axis=1, keepdims=True) * np.ones_like(x)
    inside = norm <= 1.0
    assert np.all(np.abs(y[inside]) <= a / 2 + 1e-15)       # foreground -> [-a/2, a/2]
    assert np.max(np.abs(y[inside] - 0.5 * a * x[inside])) < 1e-15
    assert np.all(np.sign(y) == np.sign(x))                  # odd, direction preserving
    # continuity at the boundary and the limit at infinity
    for u in (np.array([[1.0, 0.3, -0.2]]), np.array([[0.6, -0.8, 0.0]])):
        lo = oracle.contract(mode, a, u * (1 - 1e-9))
        hi = oracle.contract(mode, a, u * (1 + 1e-9))
        assert np.max(np.abs(lo - hi)) < 1e-8
    far = oracle.contract(mode, a, np.array([[1e12, -1e12, 3e12]]))
    if mode == 1:
        assert np.max(np.abs(np.abs(far) - 1.0)) < 1e-11
    else:
        assert abs(np.linalg.norm(far) - 1.0) < 1e-11
    # monotone in radius along a ray from the origin
    t = np.linspace(0.01, 50, 400)[:, None]
    r = np.linalg.norm(oracle.contract(mode, a, t * np.array([[0.3, -0.5, 0.81]])), axis=1)
    assert np.all(np.diff(r) > 0) if a < 2 else np.all(np.diff(r) >= -1e-15)


def test_contract_hand_values():
    # a = 0.5, x = 4: 0.5 * ((2 - 0.5)(1 - 1/4) + 0.5) = 0.5 * (1.125 + 0.5) = 0.8125
    assert oracle.contract(1, 0.5, np.array([[4.0, -4.0, 0.5]]))[0].tolist() == [0.8125, -0.8125, 0.125]
    # radial, a = 1.5, x = (0, 3, 4): ||x|| = 5, s = 0.5 * (0.5 * 0.8 + 1.5) = 0.95, y = 0.95 * (0, .6, .8)
    y = oracle.contract(2, 1.5, np.array([[0.0, 3.0, 4.0]]))[0]
    assert np.max(np.abs(y - np.array([0.0, 0.57, 0.76]))) < 1e-15


def _affine_voxel_field(A, b0, dims=(5, 6, 7)):
    """Voxel grid whose channel k holds the affine function A[k] . x + b0[k] of the
    vertex position (trilinear interpolation reproduces affine functions exactly),
    and an MLP whose density logit is h_0 (hidden layer = ReLU(h + 10) - 10 shift)."""
    H, W, D = dims
    K = len(b0)
    gx = [np.linspace(-1, 1, n) for n in dims]
    X, Y, Z = np.meshgrid(*gx, indexing="ij")
    P = np.stack([X, Y, Z], axis=-1)
    grid = [np.einsum("hwdj,kj->hwdk", P, A) + b0]
    # widths (K, K, 4): z = I h + 10 (always > 0 here), o_0 = z_0 - 10, colours from z_1
    W0 = np.eye(K)
    Wo = np.zeros((4, K))
    Wo[0, 0] = 1.0
    Wo[1:, 1 % K] = 0.5
    params = np.concatenate([W0.ravel(), np.full(K, 10.0), Wo.ravel(), np.array([-10.0, 0.0, 0.0, 0.0])])
    return oracle.Field(wl.VOXEL, grid, (K, K, 4), params)


@pytest.mark.parametrize("mode,a", [(1, 1.0), (1, 0.6), (2, 1.0)])
def test_contracted_sampling_of_an_affine_field(mode, a):
    """Per-sample density on unbounded rays equals softplus(A_0 . CC(x_j) + b_0) with
    CC taken from the textbook mip-NeRF form (a = 1) or the paper's formula typed in
    the test, and t_j = near + j Delta."""
    A = np.array([[0.7, -0.4, 0.3], [0.1, 0.2, -0.5]])
    b0 = np.array([0.2, -0.1])
    F = _affine_voxel_field(A, b0)
    F.contraction, F.contract_a = mode, a
    o = np.array([0.3, -3.0, 1.2])
    d = np.array([0.1, 0.9, -0.3])
    d /= np.linalg.norm(d)
    near, far, S = 0.05, 14.0, 23
    sigma, tau, T, w, c = oracle.trace(F, o, d, near, far, S)
    t = near + np.arange(S) * ((far - near) / (S - 1))
    x = o[None] + t[:, None] * d[None]
    if a == 1.0:
        y = 0.5 * (_mipnerf360(x) if mode == 2 else np.stack([_mipnerf360(x[:, k:k + 1])[:, 0] for k in range(3)], 1))
    else:
        n = np.abs(x)
        y = 0.5 * np.where(n <= 1, a * x, ((2 - a) * (1 - 1 / n) + a) * np.sign(x))
    z0 = y @ A[0] + b0[0]
    ref = np.log1p(np.exp(z0))
    assert np.max(np.abs(sigma - ref)) < 1e-12
    assert np.max(np.abs(np.abs(x).max(axis=1))) > 3      # the ray really leaves the cube


def test_contraction_with_a2_is_identity_inside_the_cube():
    """Per-axis CC with a = 2 is the identity on [-1,1]^3, so bounded rays render
    exactly as without contraction."""
    grid, params = tiny_field_arrays(wl.TRIPLANE, (4, 5, 6), 3, (3, 5, 4))
    o, d, near, far = tiny_rays(6, inside_start=True)
    R = oracle.Rays(o, d, near, far, 9)
    F0 = oracle.Field(wl.TRIPLANE, grid, (3, 5, 4), params)
    F2 = oracle.Field(wl.TRIPLANE, grid, (3, 5, 4), params, contraction=1, contract_a=2.0)
    a = oracle.render_forward(F0, R, np.array([0.1, 0.2, 0.3]), return_depth=True)
    b = oracle.render_forward(F2, R, np.array([0.1, 0.2, 0.3]), return_depth=True)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


# ---------------------------------------------------------------- expected depth
def _const_field(sigma, color, K=2):
    widths = [K, 4, 4]
    grid = [wl.counter_uniform(1, np.arange(3 * 3 * 3 * K, dtype=np.uint64), -1, 1).reshape(3, 3, 3, K)]
    params = np.zeros(4 * K + 4 + 4 * 4 + 4)
    params[-4] = math.log(math.expm1(sigma))
    params[-3:] = [math.log(c / (1 - c)) for c in color]
    return oracle.Field(wl.VOXEL, grid, widths, params)


def test_depth_constant_density_geometric_series():
    """depth = sum_{j=1}^R (T_{j-1} - T_j) t_j with T_j = q^{j+1}, q = e^{-Delta sigma},
    t_j = near + j Delta: (1 - q) [near S1 + Delta S2], S1 = sum_{j=1}^R q^j =
    q (1 - q^R)/(1 - q), S2 = sum_{j=1}^R j q^j = q (1 - (R+1) q^R + R q^{R+1})/(1 - q)^2."""
    sigma = 1.3
    F = _const_field(sigma, [0.3, 0.6, 0.9])
    o, d, near, far = tiny_rays(5)
    for S in (2, 9, 80):
        R = S - 1
        out, tau, depth = oracle.render_forward(F, oracle.Rays(o, d, near, far, S), None, return_depth=True)
        nr = near.astype(np.float64)
        Dl = (far.astype(np.float64) - nr) / R
        q = np.exp(-Dl * sigma)
        S1 = q * (1 - q ** R) / (1 - q)
        S2 = q * (1 - (R + 1) * q ** R + R * q ** (R + 1)) / (1 - q) ** 2
        exp = (1 - q) * (nr * S1 + Dl * S2)
        assert np.max(np.abs(depth - exp)) < 1e-12


def test_depth_is_a_weighted_mean_of_sample_depths():
    grid, params = tiny_field_arrays(wl.VOXEL, (3, 4, 5), 3, (3, 5, 4), sigma_bias=0.8)
    F = oracle.Field(wl.VOXEL, grid, (3, 5, 4), params)
    o, d, near, far = tiny_rays(6, S_list=(12,) * 6)
    S = 12
    out, tau, depth = oracle.render_forward(F, oracle.Rays(o, d, near, far, S), None, return_depth=True)
    for i in range(len(o)):
        sig, ta, T, w, c = oracle.trace(F, o[i], d[i], float(near[i]), float(far[i]), S)
        t = near[i] + np.arange(S) * ((float(far[i]) - float(near[i])) / (S - 1))
        ws = w[1:].sum()
        assert ws > 0
        mean = depth[i] / ws
        assert t[1] - 1e-12 <= mean <= t[-1] + 1e-12
        assert abs(depth[i] - np.dot(w[1:], t[1:])) < 1e-13


def _loss(F, rays, p, gt, gd, bg):
    out, tau, depth = oracle.render_forward(F, rays, bg, return_depth=True)
    return float(np.sum(p * out) + np.sum(gt * tau) + np.sum(gd * depth))


@pytest.mark.parametrize("kind,contraction", [(wl.TRIPLANE, 0), (wl.VOXEL, 1), (wl.TRIPLANE, 2)])
def test_depth_and_contraction_backward_matches_finite_differences(kind, contraction):
    """L = p.out + g_tau tau + g_depth depth on rays that leave the cube (contracted
    back into it when contraction is on): analytic gradients vs central FD."""
    dims = (4, 5, 6) if kind == wl.TRIPLANE else (3, 4, 5)
    grid, params = tiny_field_arrays(kind, dims, 3, (3, 5, 4), sigma_bias=0.4)
    F = oracle.Field(kind, grid, (3, 5, 4), params, contraction=contraction, contract_a=0.8)
    o, d, near, far = tiny_rays(6)
    far = far * (3.0 if contraction else 1.0)
    rays = oracle.Rays(o, d, near, far, 10)
    p = wl.counter_uniform(41, np.arange(18, dtype=np.uint64), -1, 1).reshape(6, 3).astype(np.float64)
    gt = wl.counter_uniform(42, np.arange(6, dtype=np.uint64), -1, 1).astype(np.float64)
    gd = wl.counter_uniform(43, np.arange(6, dtype=np.uint64), -1, 1).astype(np.float64)
    bg = np.array([0.2, 0.9, 0.5])
    gg, gp = oracle.render_backward(F, rays, p, gt, bg, grad_depth=gd)
    eps = 1e-6
    for gi, g in enumerate(F.grid):
        flat = g.reshape(-1)
        fd = np.zeros(flat.size)
        for i in range(flat.size):
            v = flat[i]
            flat[i] = v + eps
            lp = _loss(F, rays, p, gt, gd, bg)
            flat[i] = v - eps
            lm = _loss(F, rays, p, gt, gd, bg)
            flat[i] = v
            fd[i] = (lp - lm) / (2 * eps)
        assert np.max(np.abs(fd)) > 1e-3
        assert rel_inf(gg[gi].reshape(-1), fd) < 1e-6
    fd = np.zeros_like(F.params)
    for i in range(F.params.size):
        v = F.params[i]
        F.params[i] = v + eps
        lp = _loss(F, rays, p, gt, gd, bg)
        F.params[i] = v - eps
        lm = _loss(F, rays, p, gt, gd, bg)
        F.params[i] = v
        fd[i] = (lp - lm) / (2 * eps)
    assert rel_inf(gp, fd) < 1e-6
    # the depth term matters: dropping it changes the gradients
    gg0, gp0 = oracle.render_backward(F, rays, p, gt, bg)
    assert rel_inf(gp0, gp) > 1e-3


def test_depth_backward_eq3_equals_literal_derivative():
    grid, params = tiny_field_arrays(wl.TRIPLANE, (4, 5, 6), 3, (3, 5, 4), sigma_bias=0.9)
    F = oracle.Field(wl.TRIPLANE, grid, (3, 5, 4), params, contraction=1, contract_a=1.0)
    o, d, near, far = tiny_rays(6)
    rays = oracle.Rays(o, d, near, 4 * far, 12)
    p = wl.counter_uniform(51, np.arange(18, dtype=np.uint64), -1, 1).reshape(6, 3)
    gd = wl.counter_uniform(52, np.arange(6, dtype=np.uint64), -1, 1)
    a = oracle.render_backward(F, rays, p, None, None, mode=0, grad_depth=gd)
    b = oracle.render_backward(F, rays, p, None, None, mode=1, grad_depth=gd)
    for u, v in zip(a[0] + [a[1]], b[0] + [b[1]]):
        assert rel_inf(u, v) < 1e-12


# ---------------------------------------------------------------- view-dependent colour (row 1)
def _vd_field(kind=wl.TRIPLANE, dims=(4, 5, 6), K=3, hid=5, F=2, seed=61, sigma_bias=0.5, contraction=0, nh=1):
    """View-dependent field with nh hidden layers per network (nh = 2: the paper's
    3-layer g_sigma / g_v)."""
    widths = (K,) + (hid,) * nh + (4,)
    cfg = wl.Config("t", kind, 4, K, widths, 1, 1, 2, dir_freqs=F)
    grid, _ = tiny_field_arrays(kind, dims, K, widths, seed=seed)
    params = wl.make_params(cfg, seed=seed + 1, sigma_bias=sigma_bias).astype(np.float64)
    # nonzero hidden biases so that ReLU decisions vary
    params = params + 0.1 * wl.counter_uniform(seed + 2, np.arange(params.size, dtype=np.uint64), -1, 1)
    return oracle.Field(kind, grid, widths, params, contraction, 0.7, F), cfg


def test_direnc_through_a_probe_network():
    """g_v's colour logit k reads one direnc entry through an identity-like path, so
    c_k = sigmoid(sin / cos(pi 2^i d_a)) exactly (per axis, per frequency
    2^0..2^{F-1}, sin then cos)."""
    K, hid, F = 2, 4, 3
    E = 6 * F
    grid = [np.zeros((3, 3, 3, K))]
    nsig = hid * K + hid + hid + 1
    wcol_in = K + E
    p = np.zeros(nsig + hid * wcol_in + hid + 3 * hid + 3)
    Wv0 = np.zeros((hid, wcol_in))
    bv0 = np.full(hid, 10.0)                     # keep z > 0: relu is the identity (+10)
    probes = [(0, 0, "sin"), (1, 2, "cos"), (2, 1, "sin")]   # (axis, freq index, fn) -> colour 0, 1, 2
    for c, (ax, i, fn) in enumerate(probes):
        Wv0[c, K + 2 * (ax * F + i) + (0 if fn == "sin" else 1)] = 1.0
    Wv1 = np.zeros((3, hid))
    for c in range(3):
        Wv1[c, c] = 1.0
    bv1 = np.full(3, -10.0)
    p[nsig:] = np.concatenate([Wv0.ravel(), bv0, Wv1.ravel(), bv1])
    Fd = oracle.Field(wl.VOXEL, grid, (K, hid, 4), p, 0, 1.0, F)
    d = np.array([0.3, -0.5, 0.81])
    d /= np.linalg.norm(d)
    sigma, tau, T, w, col = oracle.trace(Fd, np.array([0.1, 0.2, -3.0]), d, 0.5, 5.0, 4)
    for c, (ax, i, fn) in enumerate(probes):
        v = (np.sin if fn == "sin" else np.cos)(np.pi * 2.0 ** i * d[ax])
        assert np.max(np.abs(col[:, c] - 1.0 / (1.0 + np.exp(-v)))) < 1e-13


@pytest.mark.parametrize("nh", [1, 2])
def test_density_is_view_independent(nh):
    """sigma = g_sigma(h) only: the same points traversed in opposite directions get
    the same densities (in reverse order); the colours differ."""
    Fd, _ = _vd_field(kind=wl.VOXEL, dims=(3, 4, 5), nh=nh)
    a, b = np.array([-0.7, -0.2, 0.5]), np.array([0.6, 0.4, -0.5])
    L = np.linalg.norm(b - a)
    d = (b - a) / L
    s1, _, _, _, c1 = oracle.trace(Fd, a, d, 0.0, L, 9)
    s2, _, _, _, c2 = oracle.trace(Fd, b, -d, 0.0, L, 9)
    assert np.max(np.abs(s1 - s2[::-1])) < 1e-12
    assert np.max(np.abs(c1 - c2[::-1])) > 1e-3


@pytest.mark.parametrize("kind,contraction,nh", [(wl.TRIPLANE, 0, 1), (wl.VOXEL, 1, 1), (wl.TRIPLANE, 1, 2)])
def test_view_dependent_backward_matches_finite_differences(kind, contraction, nh):
    dims = (4, 5, 6) if kind == wl.TRIPLANE else (3, 4, 5)
    F, _ = _vd_field(kind, dims, contraction=contraction, nh=nh)
    o, d, near, far = tiny_rays(6)
    rays = oracle.Rays(o, d, near, far * (2.0 if contraction else 1.0), 9)
    p = wl.counter_uniform(71, np.arange(18, dtype=np.uint64), -1, 1).reshape(6, 3).astype(np.float64)
    gt = wl.counter_uniform(72, np.arange(6, dtype=np.uint64), -1, 1).astype(np.float64)
    gd = wl.counter_uniform(73, np.arange(6, dtype=np.uint64), -1, 1).astype(np.float64)
    bg = np.array([0.2, 0.9, 0.5])
    gg, gp = oracle.render_backward(F, rays, p, gt, bg, grad_depth=gd)
    eps = 1e-6
    for gi, g in enumerate(F.grid):
        flat = g.reshape(-1)
        fd = np.zeros(flat.size)
        for i in range(flat.size):
            v = flat[i]
            flat[i] = v + eps
            lp = _loss(F, rays, p, gt, gd, bg)
            flat[i] = v - eps
            lm = _loss(F, rays, p, gt, gd, bg)
            flat[i] = v
            fd[i] = (lp - lm) / (2 * eps)
        assert np.max(np.abs(fd)) > 1e-3
        assert rel_inf(gg[gi].reshape(-1), fd) < 1e-6
    fd = np.zeros_like(F.params)
    for i in range(F.params.size):
        v = F.params[i]
        F.params[i] = v + eps
        lp = _loss(F, rays, p, gt, gd, bg)
        F.params[i] = v - eps
        lm = _loss(F, rays, p, gt, gd, bg)
        F.params[i] = v
        fd[i] = (lp - lm) / (2 * eps)
    assert rel_inf(gp, fd) < 1e-6
    a = oracle.render_backward(F, rays, p, gt, bg, mode=1, grad_depth=gd)
    for u, v in zip(gg + [gp], a[0] + [a[1]]):
        assert rel_inf(u, v) < 1e-12


def test_view_dependent_matches_torch_autograd():
    """The two networks, direnc and Eq. 1 written independently in torch fp64
    (grid_sample for h, the literal T_{j-1} - T_j weights): forward and all
    gradients agree with the oracle."""
    torch = pytest.importorskip("torch")
    K, hid, Fq = 3, 5, 2
    F, _ = _vd_field(wl.TRIPLANE, (4, 5, 6), K, hid, Fq)
    o, d, near, far = tiny_rays(6, inside_start=True)
    S = 9
    rays = oracle.Rays(o, d, near, far, S)
    p = wl.counter_uniform(74, np.arange(18, dtype=np.uint64), -1, 1).reshape(6, 3).astype(np.float64)
    out_o, _ = oracle.render_forward(F, rays, None)
    gg, gp = oracle.render_backward(F, rays, p, None, None)

    planes = [torch.tensor(g, dtype=torch.float64, requires_grad=True) for g in F.grid]
    params = torch.tensor(F.params, dtype=torch.float64, requires_grad=True)
    od, dd = torch.tensor(o, dtype=torch.float64), torch.tensor(d, dtype=torch.float64)
    Dl = (torch.tensor(far, dtype=torch.float64) - torch.tensor(near, dtype=torch.float64)) / (S - 1)
    t = torch.tensor(near, dtype=torch.float64)[:, None] + torch.arange(S, dtype=torch.float64)[None] * Dl[:, None]
    x = od[:, None, :] + t[..., None] * dd[:, None, :]

    def bil(plane, a, b):
        inp = plane.permute(2, 0, 1)[None]
        g = torch.stack([b, a], dim=-1)[None]
        return torch.nn.functional.grid_sample(inp, g, mode="bilinear", align_corners=True)[0].permute(1, 2, 0)

    h = bil(planes[0], x[..., 0], x[..., 1]) + bil(planes[1], x[..., 1], x[..., 2]) + bil(planes[2], x[..., 2], x[..., 0])
    freqs = torch.tensor([2.0 ** i for i in range(Fq)], dtype=torch.float64)
    ang = torch.pi * dd[:, :, None] * freqs[None, None, :]                  # [M][3][F]
    e = torch.stack([torch.sin(ang), torch.cos(ang)], dim=-1).reshape(len(o), 6 * Fq)
    E = 6 * Fq
    n = 0

    def take(*shape):
        nonlocal n
        cnt = int(np.prod(shape))
        v = params[n:n + cnt].reshape(*shape)
        n += cnt
        return v
    Ws0, bs0, Ws1, bs1 = take(hid, K), take(hid), take(1, hid), take(1)
    Wv0, bv0, Wv1, bv1 = take(hid, K + E), take(hid), take(3, hid), take(3)
    assert n == params.numel()
    sig = torch.nn.functional.softplus((torch.relu(h @ Ws0.T + bs0) @ Ws1.T + bs1)[..., 0])
    hv = torch.cat([h, e[:, None, :].expand(-1, S, -1)], dim=-1)
    col = torch.sigmoid(torch.relu(hv @ Wv0.T + bv0) @ Wv1.T + bv1)
    T = torch.exp(-torch.cumsum(Dl[:, None] * sig, dim=1))
    wgt = T[:, :-1] - T[:, 1:]
    out = (wgt[..., None] * col[:, 1:]).sum(1)
    assert rel_inf(out.detach().numpy(), out_o) < 1e-12
    (out * torch.tensor(p)).sum().backward()
    for a, b in zip(gg, planes):
        assert rel_inf(a, b.grad.numpy()) < 1e-10
    assert rel_inf(gp, params.grad.numpy()) < 1e-10


def test_view_dependent_relu_slack_is_zero_without_ambiguity():
    """relu_slack on a view-dependent field: buffers sized for both networks, slack >= 0,
    and zero slack when no pre-activation is ambiguous (band = 0)."""
    F, _ = _vd_field(wl.TRIPLANE, (4, 5, 6))
    o, d, near, far = tiny_rays(6)
    rays = oracle.Rays(o, d, near, far, 9)
    p = wl.counter_uniform(75, np.arange(18, dtype=np.uint64), -1, 1).reshape(6, 3)
    sg, sp = oracle.relu_slack(F, rays, p, band=1e-3)
    assert sp.shape == F.params.shape and np.all(sp >= 0) and all(np.all(g >= 0) for g in sg)
    sg0, sp0 = oracle.relu_slack(F, rays, p, band=0.0)
    assert float(np.abs(sp0).sum()) == 0.0


def _direnc(d, F):
    """direnc per S:146 in the order pinned by test_direnc_through_a_probe_network:
    per axis k, per frequency 2^i: sin(pi 2^i d_k), cos(pi 2^i d_k)."""
    e = []
    for k in range(3):
        for i in range(F):
            e += [math.sin(math.pi * 2.0 ** i * d[k]), math.cos(math.pi * 2.0 ** i * d[k])]
    return np.array(e)


@pytest.mark.parametrize("net,nh", [("sigma", 1), ("color", 1), ("sigma", 2), ("color", 2)])
def test_view_dependent_relu_slack_bounds_a_flipped_decision(net, nh):
    """The two-network slack (R29) bounds the gradient jump of a flipped decision in
    either network: put hidden unit 1 of g_sigma (or g_v, whose input is
    [h ; direnc(d)]) exactly at z = 0 on one sample, evaluate the oracle gradients
    with its bias nudged to either side (the forward does not move, ReLU'
    flips), and check |g+ - g-| <= slack elementwise. nh = 2: the paper's 3-layer
    networks, the flipped first-layer decision propagating through the second."""
    K, hid, Fq = 3, 5, 2
    Fd, _ = _vd_field(wl.TRIPLANE, (4, 5, 6), K=K, hid=hid, F=Fq, nh=nh)
    o, d, near, far = tiny_rays(2, inside_start=True)
    S = 7
    rays = oracle.Rays(o[:1], d[:1], near[:1], far[:1], S)
    p = np.array([[0.7, -0.4, 0.9]])
    gt = np.array([0.3])
    bg = np.array([0.1, 0.2, 0.3])
    Dl = (float(far[0]) - float(near[0])) / (S - 1)
    x = o[0].astype(np.float64) + (float(near[0]) + 3 * Dl) * d[0].astype(np.float64)
    h = oracle.sample(Fd, x[None])[0]
    nsig = hid * K + hid + (hid * hid + hid) * (nh - 1) + hid + 1
    if net == "sigma":
        W0, b_at, u = Fd.params[:hid * K].reshape(hid, K), hid * K, h
    else:
        E = 6 * Fq
        W0 = Fd.params[nsig:nsig + hid * (K + E)].reshape(hid, K + E)
        b_at, u = nsig + hid * (K + E), np.concatenate([h, _direnc(d[0].astype(np.float64), Fq)])
    unit = 1
    Fd.params[b_at + unit] -= float(W0[unit] @ u + Fd.params[b_at + unit])      # z = 0 at sample 3
    base = Fd.params[b_at + unit]
    res = []
    for eps in (+1e-11, -1e-11):
        Fd.params[b_at + unit] = base + eps
        res.append(oracle.render_backward(Fd, rays, p, gt, bg))
    Fd.params[b_at + unit] = base
    sg, sp = oracle.relu_slack(Fd, rays, p, gt, bg, band=1e-9)
    jump_p = np.abs(res[0][1] - res[1][1])
    assert jump_p.max() > 1e-6, "the flip must change the gradient"
    assert np.all(jump_p <= sp + 1e-9)
    for a, b, s_ in zip(res[0][0], res[1][0], sg):
        assert np.abs(a - b).max() > 0 or net == "sigma"
        assert np.all(np.abs(a - b) <= s_ + 1e-9)
    # the slack names the flipped network: the other network's parameters get none
    other = slice(nsig, None) if net == "sigma" else slice(0, nsig)
    assert float(np.abs(sp[other]).sum()) == 0.0
