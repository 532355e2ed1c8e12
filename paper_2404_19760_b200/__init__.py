"""B200-native (sm_100a) Lightplane Renderer hot path: fused forward / backward
emission-absorption ray marching over a triplane or voxel grid + tiny MLP,
behind the C ABI of include/lp.h (liblp_b200.so). See DESIGN.md.

Importing this package loads liblp_b200.so and fails loudly if it is missing.
"""
from . import _lib  # noqa: F401  (fails loudly without the native library)
from .render import (CONTRACT_NONE, CONTRACT_PER_AXIS, CONTRACT_RADIAL, TRIPLANE, VOXEL, Field, fwd_bwd_host,
                     render, render_backward, render_forward, set_l2_persist)
from .splat import (SplatGrid, SplatMlp, splat, splat_backward, splat_backward_mlp, splat_forward,
                    splat_forward_mlp, splat_mlp, splat_normalize)

__all__ = ["TRIPLANE", "VOXEL", "CONTRACT_NONE", "CONTRACT_PER_AXIS", "CONTRACT_RADIAL", "Field", "render",
           "render_forward", "render_backward", "fwd_bwd_host", "set_l2_persist", "SplatGrid", "splat",
           "splat_forward", "splat_normalize", "splat_backward", "SplatMlp", "splat_mlp", "splat_forward_mlp",
           "splat_backward_mlp"]
