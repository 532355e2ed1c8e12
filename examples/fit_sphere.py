"""Single-scene fit with image-level losses.

Target images come from an analytic scene, a ball of constant density and
colour. Its emission-absorption image has a closed form. For a ray that crosses
the ball along a chord of length L, the pixel is c (1 - e^{-sigma L}) + bg e^{-sigma L}.
A triplane field (random init) with the renderer's fused forward/backward
(paper_2404_19760_b200.render) is fit to those images with Adam on the
full-image MSE. Every step renders all pixels of a batch of views and
backpropagates through the CUDA kernels. No activation is stored per sample.

    python examples/fit_sphere.py --iters 300
"""
from __future__ import annotations

import argparse
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2404_19760_b200 as lpb  # noqa: E402
import workload as wl  # noqa: E402

RADIUS, SIGMA, COLOR, BG = 0.6, 6.0, (0.9, 0.35, 0.1), (0.05, 0.1, 0.2)


def analytic_images(o: np.ndarray, d: np.ndarray) -> np.ndarray:
    """Closed-form EA image of the ball |x| <= RADIUS: chord length from the ray-sphere roots."""
    b = np.sum(o * d, axis=1)
    c = np.sum(o * o, axis=1) - RADIUS ** 2
    disc = b * b - c
    L = np.where(disc > 0, 2.0 * np.sqrt(np.maximum(disc, 0.0)), 0.0)
    a = 1.0 - np.exp(-SIGMA * L)
    return a[:, None] * np.array(COLOR)[None] + (1.0 - a)[:, None] * np.array(BG)[None]


def fit(iters: int = 300, views: int = 16, img: int = 64, S: int = 96, res: int = 48, lr: float = 0.02,
        device: str = "cuda", seed: int = 0, log_every: int = 50):
    """Returns the list of per-step MSE losses."""
    cfg = wl.Config("fit", wl.TRIPLANE, res, 16, (16, 32, 4), views, img, S)
    o, d, near, far = wl.make_rays(cfg)
    target = torch.from_numpy(analytic_images(o.astype(np.float64), d.astype(np.float64)).astype(np.float32))
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)
    o, d, near, far, target = T(o), T(d), T(near), T(far), target.to(device)
    bg = T(np.array(BG, dtype=np.float32))
    planes = [(0.1 * torch.randn(s, generator=torch.Generator().manual_seed(seed + i))).to(device).requires_grad_()
              for i, s in enumerate(cfg.grid_shapes)]
    params = T(wl.make_mlp(cfg.widths, seed=seed + 7, sigma_bias=-2.0)).requires_grad_()
    opt = torch.optim.Adam(planes + [params], lr=lr)
    losses = []
    for it in range(iters):
        field = lpb.Field(cfg.kind, planes, cfg.widths, params)
        out, tau = lpb.render(field, o, d, near, far, S, bg)
        loss = torch.mean((out - target) ** 2)
        opt.zero_grad(set_to_none=True)
        loss.backward()
        opt.step()
        losses.append(float(loss.item()))
        if log_every and (it % log_every == 0 or it == iters - 1):
            print(f"iter {it:4d}  mse {losses[-1]:.5f}  psnr {-10 * math.log10(max(losses[-1], 1e-12)):.2f} dB")
    return losses


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=300)
    ap.add_argument("--views", type=int, default=16)
    ap.add_argument("--img", type=int, default=64)
    a = ap.parse_args()
    fit(a.iters, a.views, a.img)
