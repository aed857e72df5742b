"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NONE of the method's arithmetic (no density, no window, no
rect, no output-size rule): it only draws parameter arrays with the shapes and
value distributions of the paper's workloads. Both sides (oracle/ and the CUDA
path) receive exactly these float32 arrays.

Recipe:
  * N = m*H*W Gaussians, m = 16 ("N = m x (H x W)", P:1709 m=16).
  * mu = p + o: p is the equal-interval reference grid ("sampling N
    points at equal intervals"), read as a sqrt(m) x sqrt(m) sub-grid per LR
    pixel at ((j+1/2)/sqrt(m), (i+1/2)/sqrt(m)); o ~ U(-1/2, 1/2)^2.
  * The other properties follow the Gaussian Primary Head activations
    (sigmoid for alpha, c, sigma; tanh for rho) applied to normal
    draws:  "image"  -> raw_alpha~N(-3,1), raw_c~N(0,1), raw_sigma~N(-0.5,0.5),
                         raw_rho~N(0,0.5)
            "stress" -> every raw ~ N(0, 1.5)
  * Upstream gradient dL/dI ~ U(-1, 1).
  * Layout: SoA float32 -- alpha[n], mu[n,2]=(x,y), sigma[n,2]=(x,y), rho[n],
    color[n,3]=(r,g,b). Ragged batches concatenate images in order.
"""
from __future__ import annotations

import numpy as np

__all__ = ["reference_grid", "gaussians", "grad_out", "c2_scales", "CONFIGS", "Cloud"]

PARAM_SEED_BASE = 1000
GRAD_SEED_BASE = 2000


def reference_grid(H: int, W: int, m: int = 16) -> np.ndarray:
    """Equal-interval reference positions p, [m*H*W, 2] float64 (x, y), raster order
    (LR row, LR col, sub-row, sub-col)."""
    k = int(round(np.sqrt(m)))
    if k * k != m:
        raise ValueError("density m must be a perfect square (S:92 reading)")
    sub = (np.arange(k) + 0.5) / k
    yy = np.arange(H)[:, None, None, None] + sub[None, None, :, None]
    xx = np.arange(W)[None, :, None, None] + sub[None, None, None, :]
    yy, xx = np.broadcast_arrays(yy, xx)
    return np.stack([xx.reshape(-1), yy.reshape(-1)], axis=1).astype(np.float64)


def _sig(x):
    return 1.0 / (1.0 + np.exp(-x))


class Cloud(dict):
    """dict of float32 arrays: alpha, mu, sigma, rho, color (+ n)."""

    @property
    def n(self) -> int:
        return int(self["alpha"].shape[0])


def gaussians(H: int, W: int, m: int = 16, seed: int = 0, dist: str = "image",
              offset_range: float = 0.5) -> Cloud:
    rng = np.random.default_rng(seed)
    p = reference_grid(H, W, m)
    n = p.shape[0]
    o = rng.uniform(-offset_range, offset_range, size=(n, 2))
    if dist == "image":
        ra = rng.normal(-3.0, 1.0, n)
        rc = rng.normal(0.0, 1.0, (n, 3))
        rs = rng.normal(-0.5, 0.5, (n, 2))
        rr = rng.normal(0.0, 0.5, n)
    elif dist == "stress":
        ra = rng.normal(0.0, 1.5, n)
        rc = rng.normal(0.0, 1.5, (n, 3))
        rs = rng.normal(0.0, 1.5, (n, 2))
        rr = rng.normal(0.0, 1.5, n)
    else:
        raise ValueError(dist)
    c = Cloud(
        alpha=_sig(ra).astype(np.float32),
        mu=(p + o).astype(np.float32),
        sigma=_sig(rs).astype(np.float32),
        rho=np.tanh(rr).astype(np.float32),
        color=_sig(rc).astype(np.float32),
    )
    # tanh can round to exactly +-1 in float32 for the stress draw; keep |rho| < 1
    # (a precondition of the ABI) by nudging one ulp inward.
    c["rho"] = np.clip(c["rho"], np.nextafter(np.float32(-1), np.float32(0)),
                       np.nextafter(np.float32(1), np.float32(0))).astype(np.float32)
    c["sigma"] = np.maximum(c["sigma"], np.float32(1e-6)).astype(np.float32)
    return c


def concat(clouds) -> Cloud:
    return Cloud({k: np.concatenate([c[k] for c in clouds], axis=0) for k in
                  ("alpha", "mu", "sigma", "rho", "color")})


def grad_out(shape, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, size=shape).astype(np.float32)


def c2_scales() -> np.ndarray:
    """Per-patch scales of config C2: default_rng(0).uniform(1, 4, 16)."""
    return np.random.default_rng(0).uniform(1.0, 4.0, 16)


# BASELINE.json configs. (H, W, s) per image, LR sizes.
CONFIGS = {
    "C1": dict(images=[(48, 48, 4.0)], passes="fwd+bwd",
               desc="single 48x48 LR patch at x4 -> 192x192"),
    "C2": dict(images=[(48, 48, float(s)) for s in c2_scales()], passes="fwd+bwd",
               desc="training batch of 16 48x48 LR patches, s ~ U[1,4]"),
    "C3": dict(images=[(339, 510, 4.0)], passes="fwd",
               desc="DIV2K-val size 510x339 LR at x4 -> 2040x1356"),
    "C4": dict(images=[(45, 68, 30.0)], passes="fwd+bwd",
               desc="68x45 LR at x30 -> 2040x1350"),
    "C5": dict(images=[(170, 255, 8.0)] * 64, passes="fwd+bwd",
               desc="batch of 64 DIV2K-size 255x170 LR at x8 -> 2040x1360, row-band sharded"),
}
