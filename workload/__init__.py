"""Seeded synthetic workload generator shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no sampling, no MLP, no
compositing): it only produces inputs -- grids, MLP parameters, rays, near/far,
background colours and upstream gradients -- as plain float32 numpy arrays.
Both `oracle/` (through `tests/` and `bench.py`'s cpu_baseline) and the CUDA
path consume these arrays; neither side imports the other.

Recipe:

* Counter-based randomness: value(seed, i) = splitmix64 of (seed, i), so any
  shard or subset of a tensor reproduces exactly the same numbers.
* Cameras: V views on a Fibonacci sphere of radius 4 looking at the origin,
  up = +z (fallback +y), pinhole with 30 deg field of view, one ray per pixel
  centre (u+0.5, v+0.5), unit directions, views in index order; within a view
  rays come in 16x8-pixel tiles of four 8x4 blocks (`pixel_of`), the batching a
  renderer uses so that neighbouring rays sit in the same warp / CTA. (Rays: "M rays ... R+1 points per ray";
  pixel centres as SPEC.md S:193.)
* near/far: per-ray slab intersection with the cube [-1+1e-4, 1-1e-4]^3, so
  every sample of a hitting ray lies in the grid's domain (the paper's
  contracted setting). Misses get near = far = 0 (Delta = 0).
  Unbounded configs (near_far set, e.g. "cu") use one constant [near, far] for
  every ray and let the scene contraction map the samples into the cube.
* Grid theta: i.i.d. U(-0.5, 0.5), seed 0, per element index.
* MLP: W_l ~ U(+-1/sqrt(d_{l-1})) seed 1; hidden/colour biases 0;
  sigma bias softplus^-1(1.2) unless overridden.
* bg: U(0,1) seed 2 (parity) or zeros (throughput).
* grad_out: U(-1,1) seed 3 keyed on (global ray index, channel);
  grad_tau: U(-1,1) seed 4 keyed on global ray index (or None).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

__all__ = [
    "Config", "CONFIGS", "get_config", "counter_uniform", "make_grid",
    "make_mlp", "make_params", "n_params", "make_rays", "make_bg", "make_grad_out", "make_grad_tau", "make_features", "make_grid_grad",
    "camera_positions", "softplus_inv", "subset_indices",
]

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)

TRIPLANE = 0
VOXEL = 1


def _mix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser (Steele, Lea, Flood 2014) on a uint64 array."""
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        z = z ^ (z >> np.uint64(31))
    return z


def counter_uniform(seed: int, idx: np.ndarray, lo: float, hi: float) -> np.ndarray:
    """U(lo, hi) float32 values that depend only on (seed, idx).

    24 random mantissa bits -> the value before scaling is exact in float32.
    """
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        key = _mix64(np.uint64(seed) * _GOLDEN + _GOLDEN)
        u = _mix64(key + idx * _GOLDEN)
    u01 = (u >> np.uint64(40)).astype(np.float64) * (1.0 / (1 << 24))
    return (lo + (hi - lo) * u01).astype(np.float32)


def softplus_inv(y: float) -> float:
    """x such that log(1 + e^x) = y (used only to pick a bias value)."""
    return float(math.log(math.expm1(y)))


@dataclass(frozen=True)
class Config:
    name: str
    kind: int                 # TRIPLANE or VOXEL
    res: int                  # H = W = D
    K: int                    # grid channels
    widths: tuple             # MLP widths (K, hidden..., 1 + C)
    views: int
    img: int                  # square image side
    S: int                    # samples per ray = R + 1
    note: str = ""
    contraction: int = 0      # scene contraction of sample points (0 none, 1 per-axis, 2 radial)
    contract_a: float = 1.0   # contraction scale a
    near_far: Optional[tuple] = None   # constant (near, far) for every ray (unbounded scenes)
    op: str = "render"        # "render" (the renderer) or "splat" (the Splatter: widths unused)
    dir_freqs: int = 0        # F > 0: view-dependent colour, g_sigma(h) and g_v(h, direnc(d))
    splat_mlp: bool = False   # Splatter with g_s (Eq. 2): prior grid + MLP (dir_freqs = F of its direnc)
    ray_order: str = "tiled"  # order of the global ray index: "tiled" (pixel_of), "raster" (per view),
                              # "shuffled" (a seeded permutation of every ray of every view: NeRF-style
                              # random ray batches)

    @property
    def n_rays(self) -> int:
        return self.views * self.img * self.img

    @property
    def C(self) -> int:
        return self.widths[-1] - 1

    @property
    def grid_shapes(self) -> List[tuple]:
        H = W = D = self.res
        if self.kind == TRIPLANE:
            return [(H, W, self.K), (W, D, self.K), (D, H, self.K)]
        return [(H, W, D, self.K)]

    @property
    def grid_numel(self) -> int:
        return int(sum(int(np.prod(s)) for s in self.grid_shapes))

    @property
    def n_params(self) -> int:
        w = self.widths
        return int(sum(w[i + 1] * w[i] + w[i + 1] for i in range(len(w) - 1)))


# BASELINE.json "configs", read as in SURVEY.md §8.0 (A21-A24).
CONFIGS = {
    "c1": Config("c1", TRIPLANE, 16, 8, (8, 16, 4), 1, 64, 32,
                 "triplane 3x16x16 C=8, MLP 8->16->4, 64x64 image, 32 samples/ray"),
    "c2": Config("c2", VOXEL, 128, 16, (16, 32, 4), 1, 512, 256,
                 "voxel 128^3 C=16, MLP hidden 32, 512x512 view, 256 samples/ray"),
    "c3": Config("c3", TRIPLANE, 256, 32, (32, 64, 4), 1, 800, 512,
                 "triplane 3x256x256 C=32, MLP hidden 64, 800x800, 512 samples/ray"),
    "c4": Config("c4", TRIPLANE, 256, 32, (32, 64, 4), 128, 256, 128,
                 "triplane 3x256x256 C=32, 128 views at 256x256 (8.4M rays), 128 samples/ray"),
    "c5": Config("c5", VOXEL, 256, 32, (32, 64, 4), 64, 1024, 256,
                 "voxel 256^3 C=32, 64 views at 1024x1024, 256 samples/ray"),
    # The paper's own renderer MLP depth ("3-layer MLPs with a width of 64")
    "c3p": Config("c3p", TRIPLANE, 256, 32, (32, 64, 64, 4), 1, 800, 512,
                  "c3 with the paper's 3-layer width-64 MLP"),
    "c4p": Config("c4p", TRIPLANE, 256, 32, (32, 64, 64, 4), 128, 256, 128,
                  "c4 with the paper's 3-layer width-64 MLP"),
    # The paper's renderer setting for unbounded scenes: 160x160 triplanes,
    # 3-layer width-64 MLP, 384 points per ray, 256x256 renders, contracted coordinates
    # (per-axis, a = 1); rays run from near the camera to far behind the object.
    "cu": Config("cu", TRIPLANE, 160, 32, (32, 64, 64, 4), 16, 256, 384,
                 "unbounded scene: triplane 3x160x160 C=32, 3-layer MLP, 16 views at 256x256, "
                 "384 samples/ray, per-axis contraction a=1", contraction=1, contract_a=1.0,
                 near_far=(0.05, 12.0)),
    # View-dependent colour: sigma = g_sigma(h),
    # c = g_v(h, direnc(d)) with F = 4 direction frequencies, each network
    # with the config's hidden width (reading R29).
    "c1v": Config("c1v", TRIPLANE, 16, 8, (8, 16, 4), 1, 64, 32,
                  "c1 with view-dependent colour g_v(h, direnc(d)), F = 4", dir_freqs=4),
    "c4v": Config("c4v", TRIPLANE, 256, 32, (32, 64, 4), 128, 256, 128,
                  "c4 with view-dependent colour g_v(h, direnc(d)), F = 4", dir_freqs=4),
    # The paper's full renderer setting: view-dependent colour with
    # g_sigma and g_v each a 3-layer width-64 MLP, 160x160 triplanes, 384 points per ray,
    # 256x256 renders, per-axis contraction a = 1 (cu's scene); c4pv: c4's workload with these nets.
    "cuv": Config("cuv", TRIPLANE, 160, 32, (32, 64, 64, 4), 16, 256, 384,
                  "paper renderer setting: view-dependent g_sigma/g_v 3-layer width-64 MLPs (F = 4), "
                  "triplane 3x160x160 C=32, 16 views at 256x256, 384 samples/ray, per-axis contraction a=1",
                  contraction=1, contract_a=1.0, near_far=(0.05, 12.0), dir_freqs=4),
    "c4pv": Config("c4pv", TRIPLANE, 256, 32, (32, 64, 64, 4), 128, 256, 128,
                   "c4 with view-dependent g_sigma/g_v 3-layer width-64 MLPs (F = 4)", dir_freqs=4),
    # Splatter benchmark shape: N input feature maps lifted into a 160^3 voxel
    # grid, MLPs off; 32-channel features, 160 points per ray. N = 64 maps
    # of 128x128 pixels (the text gives neither N nor the map size: reading R28).
    "s1": Config("s1", VOXEL, 160, 32, (32, 4), 64, 128, 160,
                 "splatter: 64 feature maps of 128x128x32 into a 160^3 voxel grid, 160 points/ray", op="splat"),
    "s2": Config("s2", TRIPLANE, 160, 32, (32, 4), 64, 128, 160,
                 "splatter: 64 feature maps of 128x128x32 into 3x160x160 triplanes, 160 points/ray", op="splat"),
    # ... with the MLP g_s of Eq. 2 (v~ = g_s(v, h_prior(x), direnc(d)); 32-channel prior grid of
    # the target's shape, F = 4, hidden 64; reading R30) -- the paper's triplane Splatter
    "s1g": Config("s1g", VOXEL, 160, 32, (88, 64, 32), 64, 128, 160,
                  "splatter with g_s: 64 maps of 128x128x32 into a 160^3 voxel grid, prior 160^3x32, 160 points/ray",
                  op="splat", dir_freqs=4, splat_mlp=True),
    "s2g": Config("s2g", TRIPLANE, 160, 32, (88, 64, 32), 64, 128, 160,
                  "splatter with g_s: 64 maps of 128x128x32 into 3x160x160 triplanes, prior of the same shape, "
                  "160 points/ray", op="splat", dir_freqs=4, splat_mlp=True),
    # ... with the paper's 3-layer g_s ("3-layer MLPs with a width of 64")
    "s1gp": Config("s1gp", VOXEL, 160, 32, (88, 64, 64, 32), 64, 128, 160,
                   "splatter with the 3-layer g_s: 64 maps of 128x128x32 into a 160^3 voxel grid, prior 160^3x32, "
                   "160 points/ray", op="splat", dir_freqs=4, splat_mlp=True),
    "s2gp": Config("s2gp", TRIPLANE, 160, 32, (88, 64, 64, 32), 64, 128, 160,
                   "splatter with the 3-layer g_s: 64 maps of 128x128x32 into 3x160x160 triplanes, prior of the "
                   "same shape, 160 points/ray", op="splat", dir_freqs=4, splat_mlp=True),
}


def get_config(name: str, **overrides) -> Config:
    cfg = CONFIGS[name]
    if overrides:
        d = dict(cfg.__dict__)
        d.update(overrides)
        cfg = Config(**d)
    return cfg


def make_grid(cfg: Config, seed: int = 0, chunk: int = 1 << 24) -> List[np.ndarray]:
    """theta ~ U(-0.5, 0.5) i.i.d., channel-last, keyed on the flat element index
    (planes concatenated in xy, yz, zx order)."""
    out = []
    base = 0
    for shape in cfg.grid_shapes:
        n = int(np.prod(shape))
        arr = np.empty(n, dtype=np.float32)
        for s in range(0, n, chunk):
            e = min(n, s + chunk)
            arr[s:e] = counter_uniform(seed, np.arange(base + s, base + e, dtype=np.uint64), -0.5, 0.5)
        out.append(arr.reshape(shape))
        base += n
    return out


def make_mlp(widths: Sequence[int], seed: int = 1, sigma_bias: Optional[float] = None,
             hidden_bias_scale: float = 0.0) -> np.ndarray:
    """Packed params: W_0[w1][w0], b_0[w1], W_1[w2][w1], b_1[w2], ... (row-major out x in).

    Output unit 0 is the density logit; its bias is sigma_bias
    (default softplus^-1(1.2)); colour biases are 0.
    hidden_bias_scale > 0 draws hidden biases U(+-scale) (tests only).
    """
    if sigma_bias is None:
        sigma_bias = softplus_inv(1.2)
    parts = []
    off = 0
    for l in range(len(widths) - 1):
        fin, fout = widths[l], widths[l + 1]
        a = 1.0 / math.sqrt(fin)
        W = counter_uniform(seed, np.arange(off, off + fout * fin, dtype=np.uint64), -a, a)
        off += fout * fin
        if l < len(widths) - 2 and hidden_bias_scale > 0:
            b = counter_uniform(seed + 1000, np.arange(off, off + fout, dtype=np.uint64),
                                -hidden_bias_scale, hidden_bias_scale)
        else:
            b = np.zeros(fout, dtype=np.float32)
        off += fout
        if l == len(widths) - 2:
            b[0] = np.float32(sigma_bias)
        parts += [W.reshape(-1), b]
    return np.concatenate(parts).astype(np.float32)


def make_params(cfg: Config, seed: int = 1, sigma_bias: Optional[float] = None) -> np.ndarray:
    """The field's MLP parameters: one network (make_mlp), or for view-dependent
    configs (dir_freqs = F > 0) g_sigma with widths (K, hidden..., 1) followed by
    g_v with widths (K + 6F, hidden..., C) (reading R29)."""
    if not cfg.dir_freqs:
        return make_mlp(cfg.widths, seed=seed, sigma_bias=sigma_bias)
    w = list(cfg.widths)
    wsig = w[:-1] + [1]
    wcol = [w[0] + 6 * cfg.dir_freqs] + w[1:-1] + [w[-1] - 1]
    return np.concatenate([make_mlp(wsig, seed=seed, sigma_bias=sigma_bias),
                           make_mlp(wcol, seed=seed + 100, sigma_bias=0.0)]).astype(np.float32)


def n_params(cfg: Config) -> int:
    w = list(cfg.widths)
    if not cfg.dir_freqs:
        return cfg.n_params
    cnt = lambda ws: sum(ws[i + 1] * ws[i] + ws[i + 1] for i in range(len(ws) - 1))
    return int(cnt(w[:-1] + [1]) + cnt([w[0] + 6 * cfg.dir_freqs] + w[1:-1] + [w[-1] - 1]))


def camera_positions(views: int, radius: float = 4.0) -> np.ndarray:
    """Fibonacci-sphere camera centres (float64 [V][3])."""
    i = np.arange(views, dtype=np.float64)
    z = 1.0 - (2.0 * i + 1.0) / views
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = i * math.pi * (3.0 - math.sqrt(5.0))
    return radius * np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)


def _camera_basis(c: np.ndarray):
    fwd = -c / np.linalg.norm(c)
    up = np.array([0.0, 0.0, 1.0])
    if abs(float(fwd @ up)) > 0.999:
        up = np.array([0.0, 1.0, 0.0])
    right = np.cross(fwd, up)
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    return right, down, fwd


TILE_W, TILE_H = 16, 8


def pixel_of(pix: np.ndarray, img: int):
    """Ray order within a view: 16x8-pixel tiles in raster order of tiles; inside a
    tile, four 8x4 blocks (2 x 2) of 32 pixels, each block in raster order. So every
    128 consecutive rays form a compact 16x8 patch and every 32 an 8x4 patch
    (images whose side is not a multiple of 16 fall back to plain raster order)."""
    pix = np.asarray(pix, dtype=np.int64)
    if img % TILE_W or img % TILE_H:
        return pix // img, pix % img
    t, u = pix // (TILE_W * TILE_H), pix % (TILE_W * TILE_H)
    tiles_x = img // TILE_W
    tx, ty = t % tiles_x, t // tiles_x
    w, l = u // 32, u % 32
    col = tx * TILE_W + (w % 2) * 8 + l % 8
    row = ty * TILE_H + (w // 2) * 4 + l // 8
    return row, col


def _feistel_permute(idx: np.ndarray, n: int, seed: int = 6, rounds: int = 4) -> np.ndarray:
    """A seeded bijection of [0, n): a balanced Feistel network on the smallest even
    power-of-two domain >= n with splitmix64 round functions, cycle-walked back
    into [0, n). Any subset of indices maps independently (no table)."""
    bits = max(2, int(n - 1).bit_length())
    bits += bits & 1
    half = bits // 2
    mask = np.uint64((1 << half) - 1)
    with np.errstate(over="ignore"):
        keys = [_mix64(np.uint64(seed) * _GOLDEN + np.uint64(r + 1) * _C1) for r in range(rounds)]

    def perm(x):
        lo, hi = x & mask, x >> np.uint64(half)
        for k in keys:
            with np.errstate(over="ignore"):
                f = _mix64(lo ^ k) & mask
            lo, hi = hi ^ f, lo
        return (hi << np.uint64(half)) | lo

    x = np.asarray(idx, dtype=np.uint64).copy()
    todo = np.ones(x.shape, dtype=bool)
    while todo.any():
        x[todo] = perm(x[todo])
        todo = x >= np.uint64(n)
    return x.astype(np.int64)


def make_rays(cfg: Config, idx: Optional[np.ndarray] = None, start: int = 0,
              count: Optional[int] = None, fov_deg: float = 30.0, margin: float = 1e-4):
    """Rays for global ray indices `idx` (or the contiguous range [start, start+count)).

    Returns float32 arrays origins [n][3], dirs [n][3], near [n], far [n].
    """
    if idx is None:
        if count is None:
            count = cfg.n_rays - start
        idx = np.arange(start, start + count, dtype=np.int64)
    idx = np.asarray(idx, dtype=np.int64)
    if cfg.ray_order == "shuffled":
        idx = _feistel_permute(idx, cfg.n_rays)
    npix = cfg.img * cfg.img
    view = idx // npix
    pix = idx % npix
    if cfg.ray_order == "tiled":
        row, col = pixel_of(pix, cfg.img)
    else:
        row, col = pix // cfg.img, pix % cfg.img
    row = row.astype(np.float64)
    col = col.astype(np.float64)
    f = cfg.img / (2.0 * math.tan(math.radians(fov_deg) / 2.0))
    cx = cy = cfg.img / 2.0
    cams = camera_positions(cfg.views)
    bases = np.stack([np.stack(_camera_basis(c), axis=0) for c in cams], axis=0)  # [V][3 axes][3]
    xc = (col + 0.5 - cx) / f
    yc = (row + 0.5 - cy) / f
    B = bases[view]                                     # [n][3][3]
    d = xc[:, None] * B[:, 0] + yc[:, None] * B[:, 1] + B[:, 2]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = cams[view]
    if cfg.near_far is not None:
        near32 = np.full(len(idx), cfg.near_far[0], dtype=np.float32)
        far32 = np.full(len(idx), cfg.near_far[1], dtype=np.float32)
        return (o.astype(np.float32), d.astype(np.float32), near32, far32)
    # slab intersection with [-b, b]^3
    b = 1.0 - margin
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / d
        t1 = (-b - o) * inv
        t2 = (b - o) * inv
    tmin = np.max(np.minimum(t1, t2), axis=1)
    tmax = np.min(np.maximum(t1, t2), axis=1)
    near = np.maximum(tmin, 0.0)
    hit = tmax > near
    near = np.where(hit, near, 0.0)
    far = np.where(hit, tmax, 0.0)
    # pull [near, far] in by a relative hair so float32 rounding cannot leave the cube
    span = far - near
    near32 = np.where(hit, near + 1e-6 * span, 0.0).astype(np.float32)
    far32 = np.where(hit, far - 1e-6 * span, 0.0).astype(np.float32)
    return (o.astype(np.float32), d.astype(np.float32), near32, far32)


def make_bg(C: int = 3, seed: int = 2, zero: bool = False) -> np.ndarray:
    if zero:
        return np.zeros(C, dtype=np.float32)
    return counter_uniform(seed, np.arange(C, dtype=np.uint64), 0.0, 1.0)


def make_grad_out(idx: np.ndarray, C: int = 3, seed: int = 3) -> np.ndarray:
    idx = np.asarray(idx, dtype=np.uint64)
    e = idx[:, None] * np.uint64(C) + np.arange(C, dtype=np.uint64)[None, :]
    return counter_uniform(seed, e.reshape(-1), -1.0, 1.0).reshape(len(idx), C)


def make_features(idx: np.ndarray, K: int, seed: int = 7) -> np.ndarray:
    """Splatter input: per-pixel features U(-1,1) keyed on (global ray index, channel)."""
    idx = np.asarray(idx, dtype=np.uint64)
    e = idx[:, None] * np.uint64(K) + np.arange(K, dtype=np.uint64)[None, :]
    return counter_uniform(seed, e.reshape(-1), -1.0, 1.0).reshape(len(idx), K)


def make_grid_grad(shapes, seed: int = 8) -> List[np.ndarray]:
    """Upstream gradient of a grid-shaped output: U(-1,1) keyed on the flat element index."""
    out, base = [], 0
    for s in shapes:
        n = int(np.prod(s))
        out.append(counter_uniform(seed, np.arange(base, base + n, dtype=np.uint64), -1.0, 1.0).reshape(s))
        base += n
    return out


def make_grad_tau(idx: np.ndarray, seed: int = 4) -> np.ndarray:
    return counter_uniform(seed, np.asarray(idx, dtype=np.uint64), -1.0, 1.0)


def subset_indices(cfg: Config, n: int = 4096, seed: int = 5) -> np.ndarray:
    """The fixed parity / cpu-baseline subset: the first n/2 rays of view 0 taken
    from the image centre rows (so most of them hit the cube) plus n/2
    counter-random rays over the whole batch. Sorted, unique."""
    if n >= cfg.n_rays:
        return np.arange(cfg.n_rays, dtype=np.int64)
    half = n // 2
    npix = cfg.img * cfg.img
    first = (npix // 2 - cfg.img // 2 + np.arange(half, dtype=np.int64)) % npix
    r = counter_uniform(seed, np.arange(n - half, dtype=np.uint64), 0.0, 1.0).astype(np.float64)
    rnd = np.minimum((r * cfg.n_rays).astype(np.int64), cfg.n_rays - 1)
    allidx = np.unique(np.concatenate([first, rnd]))
    return allidx
