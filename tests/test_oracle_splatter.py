"""Pins for the oracle's Splatter:

* the unnormalised splat is the exact adjoint of the rays' gather, where the
  gather is built from oracle.sample (itself pinned against scipy's
  map_coordinates in test_oracle_pins.py) on the explicit point list;
* partition of unity: theta_weight collects exactly one unit of weight per
  in-cube sample and plane;
* constant features splat to that constant on every touched cell and exactly 0
  elsewhere ("averages the information splatted at identical positions");
* a vertex-coincident sample puts v on that vertex (SPEC's worked example);
* the backward is the exact transpose of the (linear) normalised splat:
  finite differences and the adjoint identity.
"""
import numpy as np
import pytest

import oracle
import workload as wl
from tests.helpers import rel_inf, tiny_rays


def _spec(kind, K=3, contraction=0):
    dims = (4, 5, 6) if kind == wl.TRIPLANE else (3, 4, 5)
    return oracle.GridSpec(kind, dims, K, contraction, 0.8)


def _points(rays):
    pts, owner = [], []
    for i in range(rays.n):
        span = max(rays.far[i] - rays.near[i], 0.0)
        dl = span / (rays.S - 1)
        for j in range(rays.S):
            t = rays.near[i] + j * dl
            pts.append(rays.o[i] + t * rays.d[i])
            owner.append(i)
    return np.array(pts), np.array(owner)


def _gather_rays(spec, rays, g):
    """sum_j h_g(x_ij) per ray from oracle.sample on the explicit point list."""
    F = oracle.Field(spec.kind, g, (spec.K, 2), np.zeros(spec.K * 2 + 2))   # grid only; sample() has no MLP
    x, owner = _points(rays)
    if spec.contraction:
        x = oracle.contract(spec.contraction, spec.contract_a, x)
    h = oracle.sample(F, x)
    out = np.zeros((rays.n, spec.K))
    np.add.at(out, owner, h)
    return out


@pytest.mark.parametrize("kind,contraction", [(wl.TRIPLANE, 0), (wl.VOXEL, 0), (wl.TRIPLANE, 1), (wl.VOXEL, 2)])
def test_splat_is_adjoint_of_the_rays_gather(kind, contraction):
    spec = _spec(kind, contraction=contraction)
    o, d, near, far = tiny_rays(6)
    rays = oracle.Rays(o, d, near, far * (2.5 if contraction else 1.0), 9)
    v = wl.counter_uniform(80, np.arange(6 * spec.K, dtype=np.uint64), -1, 1).reshape(6, spec.K)
    th, wt = oracle.splat_rays(spec, rays, v)
    g = [wl.counter_uniform(81 + i, np.arange(int(np.prod(s)), dtype=np.uint64), -1, 1).reshape(s).astype(np.float64)
         for i, s in enumerate(spec.shapes())]
    lhs = sum(float(np.sum(a * b)) for a, b in zip(th, g))
    rhs = float(np.sum(v * _gather_rays(spec, rays, g)))
    assert abs(lhs - rhs) < 1e-12 * max(1.0, abs(lhs))
    assert abs(lhs) > 1e-3


@pytest.mark.parametrize("kind", [wl.TRIPLANE, wl.VOXEL])
def test_splat_weights_partition_of_unity(kind):
    spec = _spec(kind)
    o, d, near, far = tiny_rays(6)
    rays = oracle.Rays(o, d, near, far, 11)
    th, wt = oracle.splat_rays(spec, rays, np.ones((6, spec.K)))
    x, _ = _points(rays)
    inside = int(np.sum(np.all(np.abs(x) <= 1.0, axis=1)))
    assert 0 < inside < len(x)                     # some samples leave the cube and splat nothing
    for w in wt:
        assert abs(float(np.sum(w)) - inside) < 1e-12
        assert np.all(w >= 0)


@pytest.mark.parametrize("kind", [wl.TRIPLANE, wl.VOXEL])
def test_constant_features_normalise_to_the_constant(kind):
    spec = _spec(kind)
    o, d, near, far = tiny_rays(6)
    rays = oracle.Rays(o, d, near, far, 13)
    c = np.array([0.25, -1.5, 3.0])
    out, th, wt = oracle.splat_forward(spec, rays, np.tile(c, (6, 1)))
    for a, w in zip(out, wt):
        touched = w[..., 0] > 0
        assert touched.any() and (~touched).any()
        assert np.max(np.abs(a[touched] - c)) < 1e-13
        assert np.all(a[~touched] == 0.0)


def test_vertex_coincident_sample():
    """One ray whose samples sit on voxel vertices: each vertex gets v exactly."""
    spec = oracle.GridSpec(wl.VOXEL, (5, 5, 5), 2)
    # vertices at x = -1, -0.5, 0, 0.5, 1 along the x axis, y = z = 0
    rays = oracle.Rays(np.array([[-1.0, 0.0, 0.0]]), np.array([[1.0, 0.0, 0.0]]), [0.0], [2.0], 5)
    v = np.array([[0.7, -0.2]])
    out, th, wt = oracle.splat_forward(spec, rays, v)
    for i in range(5):
        assert abs(wt[0][i, 2, 2, 0] - 1.0) < 1e-15
        assert np.max(np.abs(out[0][i, 2, 2] - v[0])) < 1e-15
    assert abs(float(np.sum(wt[0])) - 5.0) < 1e-15
    # backward: grad_features = sum over the ray's samples of grad_out / weight at those vertices
    g = [np.zeros((5, 5, 5, 2))]
    g[0][1, 2, 2] = [1.0, 2.0]
    gv = oracle.splat_backward(spec, rays, g, wt)
    assert np.max(np.abs(gv[0] - np.array([1.0, 2.0]))) < 1e-15


@pytest.mark.parametrize("kind,contraction", [(wl.TRIPLANE, 0), (wl.VOXEL, 1)])
def test_splat_backward_matches_finite_differences(kind, contraction):
    spec = _spec(kind, contraction=contraction)
    o, d, near, far = tiny_rays(5)
    rays = oracle.Rays(o, d, near, far * (2.0 if contraction else 1.0), 7)
    v = wl.counter_uniform(90, np.arange(5 * spec.K, dtype=np.uint64), -1, 1).reshape(5, spec.K).astype(np.float64)
    g = [wl.counter_uniform(91 + i, np.arange(int(np.prod(s)), dtype=np.uint64), -1, 1).reshape(s).astype(np.float64)
         for i, s in enumerate(spec.shapes())]

    def loss(vv):
        out, _, _ = oracle.splat_forward(spec, rays, vv)
        return sum(float(np.sum(a * b)) for a, b in zip(out, g))

    _, _, wt = oracle.splat_forward(spec, rays, v)
    gv = oracle.splat_backward(spec, rays, g, wt)
    fd = np.zeros_like(v)
    eps = 1e-6
    for idx in np.ndindex(*v.shape):
        vp, vm = v.copy(), v.copy()
        vp[idx] += eps
        vm[idx] -= eps
        fd[idx] = (loss(vp) - loss(vm)) / (2 * eps)
    assert np.max(np.abs(fd)) > 1e-2
    assert rel_inf(gv, fd) < 1e-8


# ---------------------------------------------------------------- g_s (Eq. 2)
def _identity_gs(C_in, Kp, F, K, block):
    """g_s with widths (C_in + Kp + 6F, 2K, K) whose output is one input block exactly:
    hidden = [relu(x), relu(-x)], output = hidden_+ - hidden_- (block: 'v', 'prior' or 'dir')."""
    nin = C_in + Kp + 6 * F
    off = {"v": 0, "prior": C_in, "dir": C_in + Kp}[block]
    W0 = np.zeros((2 * K, nin))
    for k in range(K):
        W0[k, off + k] = 1.0
        W0[K + k, off + k] = -1.0
    W1 = np.concatenate([np.eye(K), -np.eye(K)], axis=1)
    params = np.concatenate([W0.ravel(), np.zeros(2 * K), W1.ravel(), np.zeros(K)])
    return (nin, 2 * K, K), params


def _prior(spec, Kp, seed=95):
    return [wl.counter_uniform(seed + i, np.arange(int(np.prod(s)), dtype=np.uint64), -1, 1).reshape(s).astype(np.float64)
            for i, s in enumerate(spec.shapes(Kp))]


@pytest.mark.parametrize("kind", [wl.TRIPLANE, wl.VOXEL])
def test_gs_identity_on_features_reduces_to_the_plain_splat(kind):
    spec = _spec(kind)
    o, d, near, far = tiny_rays(6)
    rays = oracle.Rays(o, d, near, far, 9)
    v = wl.counter_uniform(96, np.arange(6 * spec.K, dtype=np.uint64), -1, 1).reshape(6, spec.K)
    widths, params = _identity_gs(spec.K, 2, 2, spec.K, "v")
    g = oracle.SplatMlp(_prior(spec, 2), widths, params, spec.K, 2)
    a = oracle.splat_forward_mlp(spec, rays, v, g)
    b = oracle.splat_forward(spec, rays, v)
    for u, w in zip(a[0] + a[1] + a[2], b[0] + b[1] + b[2]):
        assert np.max(np.abs(u - w)) < 1e-13


@pytest.mark.parametrize("kind,contraction", [(wl.TRIPLANE, 0), (wl.VOXEL, 1)])
def test_gs_reading_the_prior_splats_the_prior_samples(kind, contraction):
    """g_s = the prior block: theta = sum_ij w(x_ij) h_prior(x_ij), built independently
    from oracle.sample (scipy-pinned) and oracle.splat (adjoint-pinned) on the point list."""
    spec = _spec(kind, K=3, contraction=contraction)
    o, d, near, far = tiny_rays(6)
    rays = oracle.Rays(o, d, near, far * (2.0 if contraction else 1.0), 9)
    prior = _prior(spec, 3)
    widths, params = _identity_gs(2, 3, 1, 3, "prior")
    g = oracle.SplatMlp(prior, widths, params, 2, 1)
    v = np.zeros((6, 2))
    out, th, wt = oracle.splat_forward_mlp(spec, rays, v, g)
    x, _ = _points(rays)
    if contraction:
        x = oracle.contract(contraction, spec.contract_a, x)
    Fp = oracle.Field(kind, prior, (3, 2), np.zeros(3 * 2 + 2))
    vals = oracle.sample(Fp, x)
    ref = oracle.splat(Fp, x, vals)
    for a, b in zip(th, ref):
        assert np.max(np.abs(a - b)) < 1e-13
    assert max(np.max(np.abs(a)) for a in th) > 0.1


def test_gs_reading_direnc():
    """g_s = the direnc block (F = 1: sin(pi d_x), cos(pi d_x), sin(pi d_y)): equals the
    plain splat of those per-ray values (numpy sin / cos)."""
    spec = _spec(wl.VOXEL)
    o, d, near, far = tiny_rays(6)
    rays = oracle.Rays(o, d, near, far, 9)
    widths, params = _identity_gs(2, 2, 1, 3, "dir")
    g = oracle.SplatMlp(_prior(spec, 2), widths, params, 2, 1)
    a = oracle.splat_forward_mlp(spec, rays, np.zeros((6, 2)), g)
    dd = rays.d
    feats = np.stack([np.sin(np.pi * dd[:, 0]), np.cos(np.pi * dd[:, 0]), np.sin(np.pi * dd[:, 1])], axis=1)
    b = oracle.splat_forward(spec, rays, feats)
    for u, w in zip(a[0] + a[1], b[0] + b[1]):
        assert np.max(np.abs(u - w)) < 1e-12


@pytest.mark.parametrize("kind,nh", [(wl.TRIPLANE, 1), (wl.VOXEL, 1), (wl.TRIPLANE, 2), (wl.VOXEL, 2)])
def test_gs_backward_matches_finite_differences(kind, nh):
    """nh = 2: the paper's 3-layer g_s."""
    spec = _spec(kind, K=3)
    o, d, near, far = tiny_rays(4)
    rays = oracle.Rays(o, d, near, far, 6)
    C_in, Kp, F, hid = 2, 2, 1, 5
    widths = (C_in + Kp + 6 * F,) + (hid,) * nh + (spec.K,)
    params = wl.make_mlp(widths, seed=97, hidden_bias_scale=0.3).astype(np.float64)
    prior = _prior(spec, Kp)
    g = oracle.SplatMlp(prior, widths, params, C_in, F)
    v = wl.counter_uniform(98, np.arange(4 * C_in, dtype=np.uint64), -1, 1).reshape(4, C_in).astype(np.float64)
    gout = [wl.counter_uniform(99 + i, np.arange(int(np.prod(s)), dtype=np.uint64), -1, 1).reshape(s).astype(np.float64)
            for i, s in enumerate(spec.shapes())]
    _, _, wt = oracle.splat_forward_mlp(spec, rays, v, g)

    def loss(vv, gg):
        out, _, _ = oracle.splat_forward_mlp(spec, rays, vv, gg)
        return sum(float(np.sum(a * b)) for a, b in zip(out, gout))

    gv, gpr, gpar = oracle.splat_backward_mlp(spec, rays, v, g, gout, wt)
    eps = 1e-6
    fd = np.zeros_like(v)
    for idx in np.ndindex(*v.shape):
        vp, vm = v.copy(), v.copy()
        vp[idx] += eps
        vm[idx] -= eps
        fd[idx] = (loss(vp, g) - loss(vm, g)) / (2 * eps)
    assert rel_inf(gv, fd) < 1e-6
    fdp = np.zeros_like(params)
    for i in range(params.size):
        for sgn, store in ((1, 0), (-1, 1)):
            pp = params.copy()
            pp[i] += sgn * eps
            val = loss(v, oracle.SplatMlp(prior, widths, pp, C_in, F))
            fdp[i] += sgn * val / (2 * eps)
    assert rel_inf(gpar, fdp) < 1e-6
    for pi_, pl in enumerate(prior):
        flat = pl.reshape(-1)
        fdq = np.zeros(flat.size)
        for i in range(flat.size):
            keep = flat[i]
            flat[i] = keep + eps
            lp = loss(v, oracle.SplatMlp(prior, widths, params, C_in, F))
            flat[i] = keep - eps
            lm = loss(v, oracle.SplatMlp(prior, widths, params, C_in, F))
            flat[i] = keep
            fdq[i] = (lp - lm) / (2 * eps)
        assert rel_inf(gpr[pi_].reshape(-1), fdq) < 1e-6
    assert np.max(np.abs(gv)) > 1e-3 and max(np.max(np.abs(a)) for a in gpr) > 1e-3


@pytest.mark.parametrize("kind,nh", [(wl.TRIPLANE, 1), (wl.VOXEL, 1), (wl.TRIPLANE, 2)])
def test_gs_relu_slack_bounds_a_flipped_decision(kind, nh):
    """The g_s slack (parity metric allowance) bounds the jump of the features,
    prior and parameter gradients when one g_s ReLU decision flips: hidden
    unit 2 is put exactly at z = 0 on one sample (u = [v ; h_prior(x) ;
    direnc(d)]), the gradients are evaluated with its bias nudged to either
    side, and |g+ - g-| <= slack elementwise; band 0 gives zero slack. nh = 2:
    the paper's 3-layer g_s, the flipped first-layer decision propagating
    through the second hidden layer."""
    spec = _spec(kind, K=3)
    o, d, near, far = tiny_rays(2, inside_start=True)
    S = 6
    rays = oracle.Rays(o[:1], d[:1], near[:1], far[:1], S)
    C_in, Kp, F, hid = 2, 2, 1, 5
    widths = (C_in + Kp + 6 * F,) + (hid,) * nh + (spec.K,)
    params = wl.make_mlp(widths, seed=97, hidden_bias_scale=0.3).astype(np.float64)
    prior = _prior(spec, Kp)
    v = np.array([[0.6, -0.8]])
    gout = [wl.counter_uniform(99 + i, np.arange(int(np.prod(s)), dtype=np.uint64), -1, 1).reshape(s).astype(np.float64)
            for i, s in enumerate(spec.shapes())]
    Dl = (float(far[0]) - float(near[0])) / (S - 1)
    x = o[0].astype(np.float64) + (float(near[0]) + 2 * Dl) * d[0].astype(np.float64)
    Fp = oracle.Field(spec.kind, prior, (Kp, 2), np.zeros(Kp * 2 + 2))
    dd = d[0].astype(np.float64)
    e = [f(np.pi * dd[k]) for k in range(3) for f in (np.sin, np.cos)]          # F = 1: sin, cos per axis
    u = np.concatenate([v[0], oracle.sample(Fp, x[None])[0], e])
    In = widths[0]
    W0, b_at, unit = params[:hid * In].reshape(hid, In), hid * In, 2
    params[b_at + unit] -= float(W0[unit] @ u + params[b_at + unit])
    base = params[b_at + unit]
    g0 = oracle.SplatMlp(prior, widths, params, C_in, F)
    _, _, wt = oracle.splat_forward_mlp(spec, rays, v, g0)
    res = []
    for eps in (+1e-11, -1e-11):
        pp = params.copy()
        pp[b_at + unit] = base + eps
        res.append(oracle.splat_backward_mlp(spec, rays, v, oracle.SplatMlp(prior, widths, pp, C_in, F), gout, wt))
    sv, spr, spar = oracle.splat_mlp_relu_slack(spec, rays, v, g0, gout, wt, band=1e-9)
    jv, jpar = np.abs(res[0][0] - res[1][0]), np.abs(res[0][2] - res[1][2])
    assert jpar.max() > 1e-6 and jv.max() > 1e-6, "the flip must change the gradients"
    assert np.all(jv <= sv + 1e-9) and np.all(jpar <= spar + 1e-9)
    for a, b, s_ in zip(res[0][1], res[1][1], spr):
        assert np.all(np.abs(a - b) <= s_ + 1e-9)
    assert max(float(np.abs(a - b).max()) for a, b in zip(res[0][1], res[1][1])) > 1e-8
    z = oracle.splat_mlp_relu_slack(spec, rays, v, g0, gout, wt, band=0.0)
    assert float(np.abs(z[0]).sum() + sum(np.abs(a).sum() for a in z[1]) + np.abs(z[2]).sum()) == 0.0
