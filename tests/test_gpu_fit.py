"""End-to-end training through the fused renderer:
a triplane field fit to closed-form images of an analytic ball with Adam on the
full-image MSE; the loss must fall by 4x and stay finite."""
import math
import os
import sys

import pytest

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples"))


def test_fit_analytic_ball_loss_decreases():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from fit_sphere import fit
    losses = fit(iters=150, views=8, img=48, log_every=0)
    assert all(math.isfinite(x) for x in losses)
    assert losses[-1] < 0.25 * losses[0], (losses[0], losses[-1])
