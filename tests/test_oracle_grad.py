"""Pins of the oracle's backward pass (direct per-pair derivatives) against central finite
differences of its own forward in float64, and against closed forms.

The gradient of the truncated sum is that of the fixed pair set (reading R11): a
perturbation that moves a window edge across a pixel is skipped.
"""
import numpy as np
import pytest

import oracle as O
import gsr_synth as S

FIELDS = [("alpha", None), ("mu", 0), ("mu", 1), ("sigma", 0), ("sigma", 1), ("rho", None),
          ("color", 0), ("color", 1), ("color", 2)]


def f64(cl):
    return {k: np.array(v, np.float64) for k, v in cl.items()}


def loss(cl, H, W, s, r, g):
    return float((O.render_fwd(cl, H, W, s, r, mode="rect") * g).sum())


@pytest.mark.parametrize("H,W,m,s,r,dist,seed", [
    (3, 3, 1, 1.0, 1.0, "image", 1),
    (4, 3, 4, 1.7, 0.5, "image", 2),
    (3, 4, 4, 2.0, 0.1, "stress", 3),
    (4, 4, 1, 3.0, 0.5, "stress", 4),
    (2, 3, 4, 3.0, 1.0, "image", 5),
    (4, 3, 4, (1.7, 2.6), 0.5, "image", 6),     # scale vector (R22)
    (3, 4, 4, (3.0, 1.25), 0.1, "stress", 7),
])
def test_backward_matches_central_fd(H, W, m, s, r, dist, seed):
    cl = f64(S.gaussians(H, W, m=m, seed=seed, dist=dist))
    cl["alpha"] = np.maximum(cl["alpha"], 0.2)          # keep every term visible
    Hs, Ws = O.out_dims(H, W, s)
    g = S.grad_out((Hs, Ws, 3), seed=seed + 100).astype(np.float64)
    grads = O.render_bwd(cl, H, W, s, r, g, mode="rect")
    base_rects = O.rects(cl, H, W, s, r)
    n = cl["alpha"].shape[0]
    checked = 0
    rng = np.random.default_rng(seed)
    for i in rng.permutation(n)[:min(n, 12)]:
        for name, j in FIELDS:
            h = 1e-6
            p, q = f64(cl), f64(cl)
            if j is None:
                p[name][i] += h; q[name][i] -= h
            else:
                p[name][i, j] += h; q[name][i, j] -= h
            if name == "mu" and not (np.array_equal(O.rects(p, H, W, s, r), base_rects) and
                                     np.array_equal(O.rects(q, H, W, s, r), base_rects)):
                continue                                   # window edge moved: not differentiable
            fd = (loss(p, H, W, s, r, g) - loss(q, H, W, s, r, g)) / (2 * h)
            an = grads[name][i] if j is None else grads[name][i, j]
            scale = max(abs(fd), 1e-3 * abs(grads["alpha"][i]) + 1e-8)
            assert abs(an - fd) <= 2e-6 * scale + 1e-9, (name, j, i, an, fd)
            checked += 1
    assert checked >= 9 * min(n, 12) - 24


def test_backward_closed_forms_single_pixel():
    """With dL/dI one-hot at (y, x, k): dL/d alpha = c_k f(x/s, y/s), dL/dc_k = alpha f,
    dL/dc_j = 0 for j != k (Eq. 1). At the centre of an isotropic Gaussian the mu
    gradient vanishes and d/d sigma_x = d/d sigma_y = -alpha c_k f / sigma (d f/d sigma at the
    peak of 1/(2 pi sigma_x sigma_y))."""
    s = 2.0
    al, c = 0.6, (0.2, 0.7, 0.9)
    g1 = {"alpha": np.array([al]), "mu": np.array([[3.0, 2.5]]), "sigma": np.array([[0.8, 0.8]]),
          "rho": np.array([0.0]), "color": np.array([c])}
    H, W = 6, 6
    Hs, Ws = O.out_dims(H, W, s)
    G = np.zeros((Hs, Ws, 3))
    G[5, 6, 1] = 1.0                       # pixel (x=6, y=5) = (3, 2.5) LR: the centre
    d = O.render_bwd(g1, H, W, s, 1.0, G)
    f = 1.0 / (2 * np.pi * 0.64)
    assert d["alpha"][0] == pytest.approx(c[1] * f, rel=1e-14)
    assert d["color"][0] == pytest.approx([0.0, al * f, 0.0], rel=1e-14)
    assert abs(d["mu"][0]).max() < 1e-15
    assert d["sigma"][0] == pytest.approx([-al * c[1] * f / 0.8] * 2, rel=1e-13)
    assert d["rho"][0] == pytest.approx(0.0, abs=1e-15)


def test_backward_invalid_and_outside_get_zero():
    """R20/R10: invalid Gaussians and Gaussians whose window misses the image get zero gradient;
    pruning consistency: a Gaussian invisible in the forward gets exactly 0."""
    H, W, s, r = 4, 4, 2.0, 0.1
    cl = f64(S.gaussians(H, W, m=1, seed=0))
    cl["sigma"][0] = (0.0, 0.3)
    cl["rho"][1] = 1.0
    cl["mu"][2] = (-5.0, 1.0)
    cl["mu"][3] = (1.0, 40.0)
    Hs, Ws = O.out_dims(H, W, s)
    d = O.render_bwd(cl, H, W, s, r, np.ones((Hs, Ws, 3)))
    for i in range(4):
        for k in d:
            assert not np.any(d[k][i]), (k, i)
    assert np.any(d["alpha"][4:])


def test_backward_row_bands_sum_to_full():
    """Band decomposition: gradients are sums over pixels, so the sum of the
    per-band gradients equals the full gradient."""
    H, W, s, r = 6, 5, 2.0, 0.3
    cl = f64(S.gaussians(H, W, m=4, seed=8))
    Hs, Ws = O.out_dims(H, W, s)
    g = S.grad_out((Hs, Ws, 3), seed=1).astype(np.float64)
    full = O.render_bwd(cl, H, W, s, r, g)
    acc = {k: np.zeros_like(v) for k, v in full.items()}
    for rb, re in [(0, 4), (4, 9), (9, Hs)]:
        part = O.render_bwd(cl, H, W, s, r, g[rb:re], rows=(rb, re))
        for k in acc:
            acc[k] += part[k]
    for k in full:
        np.testing.assert_allclose(acc[k], full[k], rtol=1e-12, atol=1e-14)
    # and the forward bands concatenate to the full image
    bands = [O.render_fwd(cl, H, W, s, r, rows=(rb, re)) for rb, re in [(0, 4), (4, 9), (9, Hs)]]
    assert np.array_equal(np.concatenate(bands), O.render_fwd(cl, H, W, s, r))


def test_backward_index_subset_and_absmass():
    H, W, s, r = 5, 5, 2.0, 0.3
    cl = f64(S.gaussians(H, W, m=4, seed=12))
    Hs, Ws = O.out_dims(H, W, s)
    g = S.grad_out((Hs, Ws, 3), seed=4).astype(np.float64)
    full = O.render_bwd(cl, H, W, s, r, g, want_absmass=True)
    idx = np.array([3, 17, 50, 99])
    sub = O.render_bwd(cl, H, W, s, r, g, idx=idx, want_absmass=True)
    for k in full:
        assert np.array_equal(sub[k], full[k][idx]), k
    # |sum of terms| <= sum of |terms|
    flat = np.concatenate([full["alpha"][:, None], full["mu"], full["sigma"], full["rho"][:, None],
                           full["color"]], 1)
    assert (np.abs(flat) <= full["absmass"] * (1 + 1e-12)).all()
