"""TEST INFRASTRUCTURE ONLY -- float64 oracle of the NEXT-1 training step:
Gaussian Primary Head activations -> Eq. 4 render (the C oracle) -> L1 loss
against the HR ground truth -> gradients wrt the raw head outputs (chain rule written
out from the activation definitions; the render gradient is the C oracle's direct per-pair
derivative).

  alpha = sigmoid(raw_alpha), c = sigmoid(raw_color), sigma = sigmoid(raw_sigma)
  rho = rho_scale * tanh(raw_rho)     ("tanh ... rho in [-1, 1]"; rho_scale = 1 - eps is
                                       SPEC's rho_eps reading S:91, 1 is the paper)
  mu = ref + offset                   ("mu_i = p_i + o_i", no activation on o)
  L = mean over all output elements of |I - I_gt|
  dL/dI = sign(I - I_gt) / numel (0 at ties)
"""
from __future__ import annotations

import numpy as np

from . import oracle as O


def sigmoid(x):
    x = np.asarray(x, np.float64)
    return 1.0 / (1.0 + np.exp(-x))


def activate(raw, ref, rho_scale=1.0, fp32=False):
    """raw: dict raw_alpha[n], offset[n,2], raw_sigma[n,2], raw_rho[n], raw_color[n,3] (any
    dtype, widened to float64) -> activated cloud (float64).
    fp32=True (reading R23): the activated parameters are the render's inputs, which
    are float32 on the CUDA path: every activated value is rounded to the nearest float32, and
    mu = ref + offset is the IEEE float32 sum of the float32 ref and offset (exactly what a
    float32 addition gives); the activation derivatives of the backward stay float64."""
    f = lambda k: np.asarray(raw[k], np.float64)
    if not fp32:
        return dict(alpha=sigmoid(f("raw_alpha")), mu=np.asarray(ref, np.float64) + f("offset"),
                    sigma=sigmoid(f("raw_sigma")), rho=rho_scale * np.tanh(f("raw_rho")),
                    color=sigmoid(f("raw_color")))
    r32 = lambda x: np.asarray(x, np.float32).astype(np.float64)
    mu = (np.asarray(ref, np.float32) + np.asarray(raw["offset"], np.float32)).astype(np.float64)
    return dict(alpha=r32(sigmoid(f("raw_alpha"))), mu=mu, sigma=r32(sigmoid(f("raw_sigma"))),
                rho=r32(np.float32(rho_scale) * np.asarray(np.tanh(f("raw_rho")), np.float32)),
                color=r32(sigmoid(f("raw_color"))))


def l1_step(raw, ref, images, gts, ratio=0.1, rho_scale=1.0, sample=None, fp32=False):
    """images: list of (H, W, s, g_off, g_cnt) (s a number or a scale vector); gts: list of
    [Hs, Ws, 3] ground truths. Returns (list of rendered images, loss, dict of raw gradients).
    sample (optional): per image an array of Gaussian indices local to the image; the gradients
    are then computed for those Gaussians only (rows in the image order, concatenated), the
    images and the loss always in full. fp32: see activate (reading R23)."""
    act = activate(raw, ref, rho_scale, fp32)
    n = act["alpha"].shape[0]
    outs = []
    for (H, W, s, go, gc) in images:
        sub = {k: v[go:go + gc] for k, v in act.items()}
        outs.append(O.render_fwd(sub, H, W, s, ratio, mode="rect"))
    numel = sum(o.size for o in outs)
    loss = sum(np.abs(o - np.asarray(g, np.float64)).sum() for o, g in zip(outs, gts)) / numel
    rows = (np.arange(n) if sample is None else
            np.concatenate([go + np.asarray(sm, np.int64)
                            for (H, W, s, go, gc), sm in zip(images, sample)]))
    nr = rows.size
    d = dict(alpha=np.zeros(nr), mu=np.zeros((nr, 2)), sigma=np.zeros((nr, 2)),
             rho=np.zeros(nr), color=np.zeros((nr, 3)), absmass=np.zeros((nr, 9)))
    at = 0
    for k_img, ((H, W, s, go, gc), o, g) in enumerate(zip(images, outs, gts)):
        sub = {k: v[go:go + gc] for k, v in act.items()}
        gsign = np.sign(o - np.asarray(g, np.float64)) / numel
        idx = None if sample is None else np.asarray(sample[k_img], np.int64)
        r = O.render_bwd(sub, H, W, s, ratio, gsign, idx=idx, want_absmass=True)
        cnt = gc if idx is None else idx.size
        for k in d:
            d[k][at:at + cnt] = r[k]
        at += cnt
    raw = {k: np.asarray(v)[rows] for k, v in raw.items()}
    n = nr
    ra = np.asarray(raw["raw_alpha"], np.float64)
    rs = np.asarray(raw["raw_sigma"], np.float64)
    rr = np.asarray(raw["raw_rho"], np.float64)
    rc = np.asarray(raw["raw_color"], np.float64)
    ds = lambda x: sigmoid(x) * (1.0 - sigmoid(x))           # d sigmoid / dx
    dt = lambda x: 1.0 - np.tanh(x) ** 2                      # d tanh / dx
    jac = np.concatenate([ds(ra)[:, None], np.ones((n, 2)), ds(rs), rho_scale * dt(rr)[:, None],
                          ds(rc)], axis=1)
    grads = dict(raw_alpha=d["alpha"] * jac[:, 0], offset=d["mu"].copy(),
                 raw_sigma=d["sigma"] * jac[:, 3:5], raw_rho=d["rho"] * jac[:, 5],
                 raw_color=d["color"] * jac[:, 6:9], absmass=d["absmass"] * np.abs(jac))
    return outs, loss, grads
