"""Shared test helpers: tiny seeded problems and error metrics (no method arithmetic)."""
import math

import numpy as np

import workload as wl


def rel_inf(a, b):
    """||a - b||_inf / ||b||_inf (DESIGN.md parity metric)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    den = np.max(np.abs(b))
    if den == 0:
        return float(np.max(np.abs(a)))
    return float(np.max(np.abs(a - b)) / den)


def tiny_field_arrays(kind, dims=(4, 5, 6), K=3, widths=(3, 5, 4), seed=11, sigma_bias=0.3,
                      hidden_bias_scale=0.2):
    H, W, D = dims
    if kind == wl.TRIPLANE:
        shapes = [(H, W, K), (W, D, K), (D, H, K)]
    else:
        shapes = [(H, W, D, K)]
    grid = []
    base = 0
    for s in shapes:
        n = int(np.prod(s))
        grid.append(wl.counter_uniform(seed, np.arange(base, base + n, dtype=np.uint64), -1.0, 1.0).reshape(s))
        base += n
    params = wl.make_mlp(widths, seed=seed + 1, sigma_bias=sigma_bias, hidden_bias_scale=hidden_bias_scale)
    # make the output layer larger so colours and density vary visibly
    return grid, params


def tiny_rays(n=6, S_list=(2, 3, 5, 8, 11, 12), seed=21, inside_start=False):
    """Rays that cross the cube; some start outside it so samples leave the domain."""
    rng_o = wl.counter_uniform(seed, np.arange(3 * n, dtype=np.uint64), -1.0, 1.0).reshape(n, 3).astype(np.float64)
    rng_t = wl.counter_uniform(seed + 1, np.arange(3 * n, dtype=np.uint64), -0.5, 0.5).reshape(n, 3).astype(np.float64)
    o = 2.0 * rng_o / np.linalg.norm(rng_o, axis=1, keepdims=True)       # on a sphere of radius 2
    target = rng_t
    d = target - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    if inside_start:
        # slab intersection with [-0.99, 0.99]^3: every sample inside the cube
        b = 0.99
        t1 = (-b - o) / d
        t2 = (b - o) / d
        near = np.max(np.minimum(t1, t2), axis=1) + 1e-6
        far = np.min(np.maximum(t1, t2), axis=1) - 1e-6
        assert np.all(far > near)
    else:
        near = np.full(n, 0.2)
        far = np.full(n, 3.4)
    return o.astype(np.float32), d.astype(np.float32), near.astype(np.float32), far.astype(np.float32)


def rel_inf_slack(a, b, slack):
    """Parity error with an elementwise allowance for ambiguous ReLU decisions:
    max(|a - b| - slack, 0) / ||b||_inf."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    s = np.asarray(slack, dtype=np.float64).ravel()
    den = np.max(np.abs(b))
    num = np.max(np.maximum(np.abs(a - b) - s, 0.0))
    return float(num / den) if den > 0 else float(num)
