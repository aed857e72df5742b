"""Pins of the NEXT-1 training-step oracle (oracle/train.py): activation closed forms and a
central finite-difference check of the raw gradients of the L1 loss (fp64)."""
import numpy as np
import pytest

import gsr_synth as S
import oracle as O
from oracle import train as T


def raw_cloud(H, W, m, seed):
    rng = np.random.default_rng(seed)
    n = m * H * W
    ref = S.reference_grid(H, W, m)
    raw = dict(raw_alpha=rng.normal(-1, 1, n), offset=rng.uniform(-0.5, 0.5, (n, 2)),
               raw_sigma=rng.normal(-0.3, 0.4, (n, 2)), raw_rho=rng.normal(0, 0.5, n),
               raw_color=rng.normal(0, 1, (n, 3)))
    return raw, ref


def test_activation_closed_forms():
    """sigmoid(0) = 1/2, tanh(0) = 0, mu = p + o exactly; SPEC S:54 examples."""
    raw = dict(raw_alpha=np.array([0.0, np.log(3.0)]), offset=np.array([[0.0, 0.0], [0.25, -1.0]]),
               raw_sigma=np.array([[0.0, 0.0], [np.log(1 / 3), 0.0]]), raw_rho=np.array([0.0, np.arctanh(0.5)]),
               raw_color=np.zeros((2, 3)))
    ref = np.array([[3.5, 7.25], [1.0, 2.0]])
    a = T.activate(raw, ref)
    assert a["alpha"][0] == 0.5 and a["alpha"][1] == pytest.approx(0.75, rel=1e-15)
    assert a["sigma"][1, 0] == pytest.approx(0.25, rel=1e-15)
    assert a["rho"][0] == 0.0 and a["rho"][1] == pytest.approx(0.5, rel=1e-15)
    assert np.array_equal(a["mu"], [[3.5, 7.25], [1.25, 1.0]])
    assert (a["color"] == 0.5).all()
    assert T.activate(raw, ref, rho_scale=1 - 1e-4)["rho"][1] == pytest.approx(0.5 * (1 - 1e-4))


@pytest.mark.parametrize("s,r,rho_scale", [(2.0, 0.3, 1.0), (1.5, 0.5, 1 - 1e-4)])
def test_l1_step_gradient_matches_fd(s, r, rho_scale):
    """The raw gradients of L = mean |I - gt| equal central finite differences of the oracle's own
    loss (ground truth offset by +-0.05 from I so no sign flips under the perturbation; window
    edges held fixed by skipping perturbations that move a rect)."""
    H, W, m = 3, 4, 1
    raw, ref = raw_cloud(H, W, m, seed=3)
    n = raw["raw_alpha"].shape[0]
    imgs = [(H, W, s, 0, n)]
    act = T.activate(raw, ref, rho_scale)
    I0 = O.render_fwd(act, H, W, s, r)
    rng = np.random.default_rng(1)
    gt = I0 + rng.choice([-0.05, 0.05], size=I0.shape)
    outs, loss, g = T.l1_step(raw, ref, imgs, [gt], r, rho_scale)
    assert loss == pytest.approx(0.05, rel=1e-12)
    rects0 = O.rects(act, H, W, s, r)
    h = 1e-6
    checked = 0
    for name, cols in [("raw_alpha", None), ("offset", 0), ("offset", 1), ("raw_sigma", 0),
                       ("raw_sigma", 1), ("raw_rho", None), ("raw_color", 2)]:
        for i in range(0, n, 3):
            p = {k: np.array(v, np.float64) for k, v in raw.items()}
            q = {k: np.array(v, np.float64) for k, v in raw.items()}
            if cols is None:
                p[name][i] += h; q[name][i] -= h
            else:
                p[name][i, cols] += h; q[name][i, cols] -= h
            if name == "offset" and not (
                    np.array_equal(O.rects(T.activate(p, ref, rho_scale), H, W, s, r), rects0) and
                    np.array_equal(O.rects(T.activate(q, ref, rho_scale), H, W, s, r), rects0)):
                continue
            lp = T.l1_step(p, ref, imgs, [gt], r, rho_scale)[1]
            lq = T.l1_step(q, ref, imgs, [gt], r, rho_scale)[1]
            fd = (lp - lq) / (2 * h)
            an = g[name][i] if cols is None else g[name][i, cols]
            assert abs(an - fd) <= 1e-6 * max(abs(fd), 1e-4) + 1e-10, (name, i, an, fd)
            checked += 1
    assert checked >= 20


def test_activate_fp32_is_the_rounded_definition():
    """Reading R23: activate(fp32=True) = the float32 rounding of the fp64 activations, and mu =
    the IEEE float32 sum ref + offset (a float32 addition, exactly reproducible)."""
    rng = np.random.default_rng(5)
    n = 500
    ref = (rng.uniform(0, 48, (n, 2))).astype(np.float32)
    raw = dict(raw_alpha=rng.normal(-3, 1, n), offset=rng.uniform(-0.5, 0.5, (n, 2)),
               raw_sigma=rng.normal(-0.5, 0.5, (n, 2)), raw_rho=rng.normal(0, 0.5, n),
               raw_color=rng.normal(0, 1, (n, 3)))
    raw = {k: v.astype(np.float32) for k, v in raw.items()}
    a64 = T.activate(raw, ref, 1.0)
    a32 = T.activate(raw, ref, 1.0, fp32=True)
    for k in ("alpha", "sigma", "rho", "color"):
        assert np.array_equal(a32[k], a64[k].astype(np.float32).astype(np.float64)), k
    mu = np.empty((n, 2), np.float32)
    np.add(ref, raw["offset"], out=mu)
    assert np.array_equal(a32["mu"], mu.astype(np.float64))
    assert np.abs(a32["mu"] - a64["mu"]).max() > 0           # the rounding is real
