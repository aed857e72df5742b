"""gsr-b200: B200-native (sm_100a) differentiable scale-aware 2D Gaussian rasterization of
GSASR (arXiv 2501.06838, Eq. 1-4 / Alg. 1), behind the C-ABI in include/gsr.h.

    from paper_2501_06838_b200 import render
    img = render(alpha, mu, sigma, rho, color, H, W, scale)   # [floor(sH), floor(sW), 3]
"""
from ._lib import GsrError, load, out_dims, tile_shape, version
from .ops import (Image, Layout, finalize_grads, finalize_grads_subset, layout, pair_count,
                  render, render_batch, render_bwd, render_bwd_batched,
                  render_bwd_moments_batched, render_bwd_moments_subset, render_fwd,
                  render_fwd_batched, render_fwd_subset, subset_workspace_for, StreamedFwdBwd,
                  TrainStepGraph, train_step_l1, validate_params)

__all__ = ["GsrError", "load", "out_dims", "tile_shape", "version", "Image", "Layout",
           "finalize_grads", "layout", "pair_count", "render", "render_batch", "render_bwd",
           "render_bwd_batched", "render_bwd_moments_batched", "render_fwd", "render_fwd_batched",
           "StreamedFwdBwd", "TrainStepGraph", "train_step_l1", "render_fwd_subset",
           "render_bwd_moments_subset", "finalize_grads_subset", "subset_workspace_for",
           "validate_params"]
