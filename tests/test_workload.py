"""Input generator checks (host logic; -m "not gpu")."""
import numpy as np

import workload as wl


def test_counter_rng_is_subset_stable_and_uniform():
    idx = np.arange(100000, dtype=np.uint64)
    a = wl.counter_uniform(3, idx, -1, 1)
    sub = np.array([5, 77, 99999, 31337], dtype=np.uint64)
    assert np.array_equal(wl.counter_uniform(3, sub, -1, 1), a[sub.astype(np.int64)])
    assert a.min() >= -1 and a.max() < 1
    assert abs(float(a.mean())) < 0.01 and abs(float(a.var()) - 1 / 3) < 0.01
    assert not np.array_equal(a, wl.counter_uniform(4, idx, -1, 1))


def test_rays_unit_and_inside_cube():
    cfg = wl.get_config("c4")
    idx = wl.subset_indices(cfg, 4096)
    o, d, near, far = wl.make_rays(cfg, idx)
    assert np.max(np.abs(np.linalg.norm(d.astype(np.float64), axis=1) - 1)) < 1e-6
    hit = far > near
    assert hit.mean() > 0.5
    for t in (near, far, 0.5 * (near + far)):
        x = o.astype(np.float64) + t[:, None].astype(np.float64) * d
        assert np.all(np.abs(x[hit]) <= 1.0)
    assert np.all(near[~hit] == 0) and np.all(far[~hit] == 0)
    # shards reproduce the full batch
    o2, d2, n2, f2 = wl.make_rays(cfg, start=int(idx[3]), count=1)
    assert np.array_equal(o2[0], o[3]) and np.array_equal(d2[0], d[3]) and n2[0] == near[3]


def test_config_sizes_match_survey():
    c = wl.CONFIGS
    assert c["c1"].grid_numel * 4 == 24576 and c["c1"].n_params == 212
    assert c["c2"].grid_numel * 4 == 134217728 and c["c2"].n_params == 676
    assert c["c3"].grid_numel * 4 == 25165824 and c["c3"].n_params == 2372
    assert c["c3p"].n_params == 6532
    assert c["c4"].n_rays == 8388608 and c["c5"].n_rays == 67108864
    assert c["c5"].grid_numel * 4 == 2 ** 31


def test_mlp_init_layout():
    p = wl.make_mlp((32, 64, 4))
    assert p.shape == (2372,)
    W0 = p[:2048]
    assert np.max(np.abs(W0)) <= 1 / np.sqrt(32)
    b1 = p[-4:]
    assert abs(np.log1p(np.exp(b1[0])) - 1.2) < 1e-6 and np.all(b1[1:] == 0)


def test_tiled_pixel_order_is_a_permutation():
    for img in (64, 256, 800):
        pix = np.arange(img * img)
        r, c = wl.pixel_of(pix, img)
        assert len(set((r * img + c).tolist())) == img * img
        assert r.min() == 0 and r.max() == img - 1 and c.max() == img - 1
    r, c = wl.pixel_of(np.arange(32), 256)     # first warp = 8x4 block
    assert set(r.tolist()) == {0, 1, 2, 3} and set(c.tolist()) == set(range(8))


def test_ray_orders_are_permutations_of_the_same_rays():
    """raster / shuffled orders (bench --ray-order) reorder the tiled batch's rays:
    same multiset of (origin, direction, near, far); the shuffle is a bijection."""
    n = 4096
    for m in (100, n, 8388608):
        x = wl._feistel_permute(np.arange(min(m, 1 << 16)), m)
        assert len(np.unique(x)) == len(x) and x.min() >= 0 and x.max() < m
    x = wl._feistel_permute(np.arange(n), n)
    assert sorted(x.tolist()) == list(range(n)) and not np.array_equal(x, np.arange(n))
    key = lambda r: sorted(map(tuple, np.concatenate([r[0], r[1], r[2][:, None], r[3][:, None]], 1).tolist()))
    ref = key(wl.make_rays(wl.get_config("c1")))
    for order in ("raster", "shuffled"):
        c = wl.get_config("c1", ray_order=order)
        rays = wl.make_rays(c)
        assert key(rays) == ref, order
        if order == "shuffled":   # any subset maps independently (no table)
            sub = wl.make_rays(c, idx=np.array([5, 77, 4000]))
            assert np.array_equal(sub[1], rays[1][[5, 77, 4000]])
