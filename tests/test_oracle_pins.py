"""Pins of the float64 oracle against what the paper and mathematics fix (CPU only).

None of these retype the oracle's formula: each checks a consequence that a
plausible mistake (dropped normalisation, sigma vs sigma^2, wrong rho sign,
x/y swap, wrong sample point, wrong window axis, off-by-one in the rect) would
break. Citations: P:<line> = /root/reference/PAPER.md (read at authoring time).
"""
import math
from pathlib import Path

import numpy as np
import pytest

import oracle as O
import gsr_synth as S

GOLD = Path(__file__).resolve().parent / "golden"


def one(alpha=1.0, mu=(0.0, 0.0), sigma=(1.0, 1.0), rho=0.0, color=(1.0, 1.0, 1.0)):
    return dict(alpha=np.array([alpha], np.float64), mu=np.array([mu], np.float64),
                sigma=np.array([sigma], np.float64), rho=np.array([rho], np.float64),
                color=np.array([color], np.float64))


def cat(*cl):
    return {k: np.concatenate([c[k] for c in cl]) for k in cl[0]}


# --------------------------------------------------------------------------- Eq. 2 closed forms
def test_eq2_closed_forms_golden():
    """Eq. 1-2 at single points; values derived by hand in the golden file."""
    rows = [l.split() for l in (GOLD / "eq2_closed_forms.txt").read_text().splitlines()
            if l.strip() and not l.startswith("#")]
    assert len(rows) >= 6
    for r in rows:
        sx, sy, rho, dx, dy, al, c, want = map(float, r)
        g = one(alpha=al, mu=(3.0, 4.0), sigma=(sx, sy), rho=rho, color=(c, c, c))
        got = O.field(g, 1e9, 1e9, np.array([[3.0 + dx, 4.0 + dy]]))
        np.testing.assert_allclose(got[0], [want] * 3, rtol=1e-14, atol=0)


# --------------------------------------------------------------------------- Poisson summation
@pytest.mark.parametrize("s", [1.0, 2.0, 2.7, 4.0])
@pytest.mark.parametrize("sig,rho", [((0.9, 0.6), 0.4), ((0.7, 1.1), -0.65), ((1.0, 1.0), 0.0)])
def test_poisson_summation_moments(s, sig, rho):
    """Eq. 4 samples the continuous Gaussian on a grid of spacing 1/s. By Poisson
    summation, for a Gaussian far from the borders and untruncated, (1/s^2) sum_pixels I equals
    alpha*c, its first moments equal mu and its central second moments equal
    [[sx^2, rho sx sy], [rho sx sy, sy^2]] up to ~exp(-2 pi^2 s^2 lambda_min) (here < 1e-12).
    Pins: the 1/(2 pi sx sy sqrt(1-rho^2)) factor, sigma vs sigma^2, the sign of rho, which
    sigma goes with x, and the sample point x/s."""
    H, W = 24, 20
    mu = (W / 2 + 0.37, H / 2 - 0.21)
    g = one(alpha=0.75, mu=mu, sigma=sig, rho=rho, color=(1.0, 0.5, 0.25))
    lam_min = min(np.linalg.eigvalsh([[sig[0] ** 2, rho * sig[0] * sig[1]],
                                      [rho * sig[0] * sig[1], sig[1] ** 2]]))
    if s * s * lam_min < 1.0:
        pytest.skip("grid too coarse for the Poisson bound")
    I = O.render_fwd(g, H, W, s, r=1.0, mode="none")
    Hs, Ws = I.shape[:2]
    Y, X = np.meshgrid(np.arange(Hs) / s, np.arange(Ws) / s, indexing="ij")
    w = I[..., 0] / s ** 2           # alpha*c_r*f/s^2, c_r = 1
    np.testing.assert_allclose(I[..., 1], 0.5 * I[..., 0], rtol=1e-15)
    np.testing.assert_allclose(I[..., 2], 0.25 * I[..., 0], rtol=1e-15)
    eps = math.exp(-2 * math.pi ** 2 * s * s * lam_min)   # Poisson aliasing bound
    tol0, tol = max(1e-11, 10 * eps), max(1e-9, 1e3 * eps)
    m0 = w.sum()
    assert abs(m0 - 0.75) < tol0
    mx, my = (w * X).sum() / m0, (w * Y).sum() / m0
    assert abs(mx - mu[0]) < tol and abs(my - mu[1]) < tol
    cxx = (w * (X - mu[0]) ** 2).sum() / m0
    cyy = (w * (Y - mu[1]) ** 2).sum() / m0
    cxy = (w * (X - mu[0]) * (Y - mu[1])).sum() / m0
    assert abs(cxx - sig[0] ** 2) < tol
    assert abs(cyy - sig[1] ** 2) < tol
    assert abs(cxy - rho * sig[0] * sig[1]) < tol


# --------------------------------------------------------------------------- window / Alg. 1
def test_window_truncation_bound():
    """Alg. 1 drops a pair only when |X-mu_x| >= rW or |Y-mu_y| >= rH. For such a point the
    Mahalanobis form satisfies Q >= h^2/lambda_max with h = min(rW, rH), so every dropped term is at
    most alpha c K exp(-h^2/(2 lambda_max)) and I_r <= I_inf <= I_r + that sum (alpha, c >= 0)."""
    H, W, s, r = 10, 12, 2.0, 0.15
    cl = S.gaussians(H, W, m=4, seed=7, dist="image")
    cl["sigma"] = (cl["sigma"] * 1.6).astype(np.float32)      # make truncation material
    Ir = O.render_fwd(cl, H, W, s, r, mode="rect")
    Iinf = O.render_fwd(cl, H, W, s, r, mode="none")
    sx = cl["sigma"][:, 0].astype(np.float64); sy = cl["sigma"][:, 1].astype(np.float64)
    rho = cl["rho"].astype(np.float64)
    lam_max = np.array([max(np.linalg.eigvalsh([[a * a, p * a * b], [p * a * b, b * b]]))
                        for a, b, p in zip(sx, sy, rho)])
    K = 1.0 / (2 * np.pi * sx * sy * np.sqrt(1 - rho ** 2))
    h = min(r * W, r * H)
    per = cl["alpha"][:, None].astype(np.float64) * cl["color"].astype(np.float64) * \
        (K * np.exp(-h * h / (2 * lam_max)))[:, None]
    bound = per.sum(axis=0)
    diff = Iinf - Ir
    assert (diff >= -1e-15).all()
    assert (diff <= bound[None, None, :] + 1e-15).all()
    assert diff.max() > 1e-6            # the test is not vacuous


def test_truncation_negligible_regime():
    """S:129 corollary of the bound above: sigma <= 0.5 and r min(H,W) >= 6 => |I_r - I_1| < 1e-6."""
    H, W, s = 30, 32, 1.5
    cl = S.gaussians(H, W, m=1, seed=3)
    cl["sigma"] = np.minimum(cl["sigma"], 0.5).astype(np.float32)
    a = O.render_fwd(cl, H, W, s, 0.2, mode="rect")
    b = O.render_fwd(cl, H, W, s, 1.0, mode="rect")
    assert np.abs(a - b).max() < 1e-6


def test_window_axis_pairing_and_strictness():
    """Reading R1/R2: half-extent r*W along x and r*H along y (x <-> W), strict '<'. A Gaussian
    placed so that a pixel sits exactly on the x edge must exclude it; rect mode must agree."""
    H, W, s, r = 8, 16, 2.0, 0.25       # hx = 4 LR px, hy = 2 LR px
    g = one(mu=(6.0, 4.0), sigma=(3.0, 3.0))
    I = O.render_fwd(g, H, W, s, r, mode="brute")
    nz = np.argwhere(I[..., 0] > 0)
    ys, xs = nz[:, 0], nz[:, 1]
    # |x/2 - 6| < 4  <=> 4 < x < 20 ;  |y/2 - 4| < 2 <=> 4 < y < 12
    assert xs.min() == 5 and xs.max() == 19
    assert ys.min() == 5 and ys.max() == 11
    R = O.rects(g, H, W, s, r)[0]
    assert tuple(R[2:]) == (5, 19, 5, 11)
    assert np.array_equal(I, O.render_fwd(g, H, W, s, r, mode="rect"))


def test_output_size_floor():
    """Reading R4: output is floor(sH) x floor(sW) (Alg. 1 l.1 'sH x sW')."""
    assert O.out_dims(48, 48, 4.0) == (192, 192)
    assert O.out_dims(339, 510, 4.0) == (1356, 2040)
    assert O.out_dims(45, 68, 30.0) == (1350, 2040)
    assert O.out_dims(10, 7, 2.5) == (25, 17)
    assert O.out_dims(7, 3, 1.5) == (10, 4)


def test_sample_point_no_half_pixel():
    """Reading R3: pixel (x, y) samples the field at (x/s, y/s) (Eq. 4). A Gaussian at
    mu = (2, 3) must peak exactly at HR pixel (2s, 3s) and be symmetric around it."""
    s = 3.0
    g = one(mu=(2.0, 3.0), sigma=(0.5, 0.5))
    I = O.render_fwd(g, 8, 8, s, 1.0, mode="brute")[..., 0]
    y, x = np.unravel_index(np.argmax(I), I.shape)
    assert (x, y) == (6, 9)
    np.testing.assert_allclose(I[9, 6 + 1:6 + 4], I[9, 6 - 1:6 - 4:-1], rtol=1e-15)
    np.testing.assert_allclose(I[9 + 1:9 + 4, 6], I[9 - 1:9 - 4:-1, 6], rtol=1e-15)


# --------------------------------------------------------------------------- invariances
@pytest.mark.parametrize("lam", [(1 / 20, 1 / 14), (3.0, 0.5)])
def test_coordinate_normalisation_invariance(lam):
    """Scale-invariance under coordinate normalisation (north_star): rescaling every length
    along x by lx and along y by ly (mu, sigma, sample points, window half-extents; rho fixed)
    turns the field into I / (lx ly) -- f is a density, Eq. 2. lam=(1/W, 1/H) is the normalised
    [0,1] frame."""
    H, W, s, r = 14, 20, 2.5, 0.1
    cl = S.gaussians(H, W, m=4, seed=11)
    lx, ly = lam
    Hs, Ws = O.out_dims(H, W, s)
    rng = np.random.default_rng(5)
    pts = np.stack([rng.uniform(0, W, 400), rng.uniform(0, H, 400)], 1)
    a = O.field(cl, r * W, r * H, pts)
    cl2 = dict(cl)
    cl2["mu"] = cl["mu"].astype(np.float64) * np.array([lx, ly])
    cl2["sigma"] = cl["sigma"].astype(np.float64) * np.array([lx, ly])
    b = O.field(cl2, r * W * lx, r * H * ly, pts * np.array([lx, ly]))
    np.testing.assert_allclose(b * (lx * ly), a, rtol=1e-12, atol=1e-300)
    # and render() is the field sampled at (x/s, y/s) with half-extents (rW, rH)
    Y, X = np.meshgrid(np.arange(Hs) / s, np.arange(Ws) / s, indexing="ij")
    f = O.field(cl, r * W, r * H, np.stack([X.ravel(), Y.ravel()], 1)).reshape(Hs, Ws, 3)
    np.testing.assert_allclose(O.render_fwd(cl, H, W, s, r, mode="brute"), f, rtol=1e-15,
                               atol=0)


@pytest.mark.parametrize("s,k", [(1.0, 2), (1.0, 4), (1.5, 2), (2.0, 3)])
def test_integer_scale_consistency(s, k):
    """Eq. 4: pixel (k x, k y) at scale k s samples (kx/(ks), ky/(ks)) = (x/s, y/s), the same
    point as pixel (x, y) at scale s, with the same window test (r W in LR units), so
    I_{ks}[k y, k x] == I_s[y, x] bit-for-bit in brute mode."""
    H, W, r = 6, 7, 0.3
    cl = S.gaussians(H, W, m=4, seed=2)
    a = O.render_fwd(cl, H, W, s, r, mode="brute")
    b = O.render_fwd(cl, H, W, k * s, r, mode="brute")
    Hs, Ws = a.shape[:2]
    assert np.array_equal(b[::k, ::k][:Hs, :Ws], a)


def test_linearity_and_empty():
    """Eq. 3/4 are plain sums: I(A u B) = I(A) + I(B); the empty cloud renders zeros."""
    H, W, s, r = 8, 9, 2.0, 0.2
    A = S.gaussians(H, W, m=1, seed=1)
    B = S.gaussians(H, W, m=4, seed=2)
    AB = {k: np.concatenate([A[k], B[k]]) for k in A}
    np.testing.assert_allclose(O.render_fwd(AB, H, W, s, r),
                               O.render_fwd(A, H, W, s, r) + O.render_fwd(B, H, W, s, r),
                               rtol=1e-13, atol=1e-300)
    E = {k: v[:0] for k, v in A.items()}
    assert not O.render_fwd(E, H, W, s, r).any()


def test_reflection_symmetries():
    """Eq. 2 symmetries: rho = 0 gives mirror symmetry about the centre; in general the
    density is point-symmetric, and (rho, dy) -> (-rho, -dy) leaves it unchanged."""
    s = 2.0
    mu = (5.0, 6.0)     # HR pixel (10, 12) is the centre
    a = O.render_fwd(one(mu=mu, sigma=(0.8, 1.3), rho=0.0), 12, 12, s, 1.0, mode="brute")[..., 0]
    np.testing.assert_allclose(a[12, 11:20], a[12, 9:0:-1], rtol=1e-15)
    b = O.render_fwd(one(mu=mu, sigma=(0.8, 1.3), rho=0.55), 12, 12, s, 1.0, mode="brute")[..., 0]
    c = O.render_fwd(one(mu=mu, sigma=(0.8, 1.3), rho=-0.55), 12, 12, s, 1.0, mode="brute")[..., 0]
    for dy in range(-4, 5):
        for dx in range(-4, 5):
            assert b[12 + dy, 10 + dx] == pytest.approx(b[12 - dy, 10 - dx], rel=1e-14)
            assert b[12 + dy, 10 + dx] == pytest.approx(c[12 - dy, 10 + dx], rel=1e-14)
    # correlation direction: rho > 0 puts mass on the (+,+) diagonal (cov_xy = rho sx sy > 0)
    assert b[14, 12] > b[14, 8]


def test_invalid_gaussians_contribute_nothing():
    """Reading R20: non-finite fields, sigma <= 0 or |rho| >= 1 make a Gaussian invalid."""
    H, W, s, r = 5, 5, 2.0, 0.5
    base = one(mu=(2.0, 2.0), sigma=(0.5, 0.5))
    ref = O.render_fwd(base, H, W, s, r)
    for k, v in [("sigma", (0.0, 0.5)), ("sigma", (0.5, -1.0)), ("rho", 1.0), ("rho", -1.0),
                 ("alpha", np.nan), ("mu", (np.inf, 2.0)), ("color", (1.0, np.nan, 1.0))]:
        bad = one(mu=(2.5, 2.5), sigma=(0.5, 0.5))
        bad[k] = np.array([v], np.float64)
        got = O.render_fwd(cat(base, bad), H, W, s, r)
        assert np.array_equal(got, ref), k
        R = O.rects(bad, H, W, s, r)[0]
        assert R[2] > R[3]


# --------------------------------------------------------------------------- brute vs rect
@pytest.mark.parametrize("cfg", [(8, 8, 4.0, 0.1, "image", 1), (6, 10, 2.5, 0.1, "stress", 2),
                                 (7, 5, 1.0, 0.5, "image", 3), (5, 5, 3.3, 1.0, "stress", 4),
                                 (4, 6, 17.0, 0.1, "image", 5),
                                 (6, 7, (2.0, 3.5), 0.2, "image", 6),
                                 (5, 8, (4.25, 1.5), 0.1, "stress", 7)])
def test_brute_equals_rect_bitwise(cfg):
    """The integer rect (R2) selects exactly the pairs of the literal predicate and the per-pixel
    sum order is ascending i in both modes, so the results are bit-identical."""
    H, W, s, r, dist, seed = cfg
    cl = S.gaussians(H, W, m=4, seed=seed, dist=dist, offset_range=1.5)
    a = O.render_fwd(cl, H, W, s, r, mode="brute")
    b = O.render_fwd(cl, H, W, s, r, mode="rect")
    assert np.array_equal(a, b)
    g = S.grad_out(a.shape, seed=3)
    ga = O.render_bwd(cl, H, W, s, r, g, mode="brute")
    gb = O.render_bwd(cl, H, W, s, r, g, mode="rect")
    for k in ga:
        assert np.array_equal(ga[k], gb[k]), k


@pytest.mark.parametrize("cfg", [(8, 9, 4.0, 0.1, "image", 11), (6, 7, 2.7, 1.0, "stress", 12),
                                 (5, 8, (3.0, 1.75), 0.2, "image", 13),
                                 (4, 6, 1.0, 1.0, "image", 14)])
def test_render_pixels_equals_brute_render(cfg):
    """gsr_oracle_render_pixels (Eq. 4 at an explicit pixel list, literal Alg. 1
    predicate P:1385) is the checker of the full-size sampled parity tests; it must equal the
    brute-mode full render bit for bit at every pixel, in any pixel order, including a scale
    vector (R22) and r = 1 (every window covers the frame)."""
    H, W, s, r, dist, seed = cfg
    cl = S.gaussians(H, W, m=4, seed=seed, dist=dist, offset_range=1.5)
    full = O.render_fwd(cl, H, W, s, r, mode="brute")
    Hs, Ws = full.shape[:2]
    ys, xs = np.meshgrid(np.arange(Hs), np.arange(Ws), indexing="ij")
    perm = np.random.default_rng(seed).permutation(Hs * Ws)
    got = O.render_pixels(cl, H, W, s, r, xs.reshape(-1)[perm], ys.reshape(-1)[perm])
    assert np.array_equal(got, full.reshape(-1, 3)[perm])
    assert np.abs(full).max() > 0


def test_pair_count_full_window():
    """r = 1 with every mu inside the frame: every Gaussian's window covers the whole image, so
    P = N * Hs * Ws."""
    H, W, s = 5, 6, 3.0
    cl = S.gaussians(H, W, m=4, seed=0, offset_range=0.2)
    Hs, Ws = O.out_dims(H, W, s)
    assert O.pair_count(cl, H, W, s, 1.0) == cl["alpha"].shape[0] * Hs * Ws


def test_pair_count_matches_nonzero_support():
    H, W, s, r = 6, 6, 2.0, 0.2
    cl = S.gaussians(H, W, m=4, seed=4)
    R = O.rects(cl, H, W, s, r)
    manual = int(sum(max(0, x1 - x0 + 1) * max(0, y1 - y0 + 1) for _, _, x0, x1, y0, y1 in R))
    assert O.pair_count(cl, H, W, s, r) == manual


# --------------------------------------------------------------------------- binning brute force
@pytest.mark.parametrize("tw,th", [(16, 16), (32, 8), (7, 5)])
def test_tile_lists_brute_vs_rect_enumeration(tw, th):
    """The brute-force binning (O(N * tiles) intersection tests) equals enumerating, for each
    Gaussian, the tiles its integer rect covers."""
    H, W, s, r = 12, 14, 3.0, 0.1
    cl = S.gaussians(H, W, m=4, seed=9, offset_range=2.0)
    counts, ids = O.tile_lists(cl, H, W, s, r, tw, th)
    Hs, Ws = O.out_dims(H, W, s)
    ntx = -(-Ws // tw)
    lists = {}
    for i, (_, _, x0, x1, y0, y1) in enumerate(O.rects(cl, H, W, s, r)):
        if x0 > x1 or y0 > y1:
            continue
        for ty in range(y0 // th, y1 // th + 1):
            for tx in range(x0 // tw, x1 // tw + 1):
                lists.setdefault(ty * ntx + tx, []).append(i)
    off = np.concatenate([[0], np.cumsum(counts)])
    for t in range(len(counts)):
        assert list(ids[off[t]:off[t + 1]]) == lists.get(t, []), t


# --------------------------------------------------------------------------- R21 support rect
def test_support_rect_closed_form():
    """Reading R21: support rect = window rect (R2) cut to the integer box
    [floor(s(mu - 13.5 sigma)), ceil(s(mu + 13.5 sigma))]. Hand-derived (float32 inputs):
    mu = (10.3, 7.7), s = 4, H = W = 32.
      sigma = (0.4, 0.25), r = 0.5: window x: floor(4(10.3 - 16)) + 1 = -22 (clip 0),
        ceil(4 * 26.3) - 1 = 105; box x: floor(4 * 4.9) = 19, ceil(4 * 15.7) = 63 -> [19, 63];
        window y: -33 (clip 0) .. ceil(4 * 23.7) - 1 = 94; box y: floor(4 * 4.325) = 17, ceil(4 * 11.075) = 45.
      sigma = (2, 3), r = 0.1: box wider than the window -> the window rect
        x: floor(4 * 7.1) + 1 = 29, ceil(4 * 13.5000002) - 1 = 54; y: 18 .. 43."""
    g = one(mu=(10.3, 7.7), sigma=(0.4, 0.25))
    g = {k: v.astype(np.float32) for k, v in g.items()}
    assert list(O.rects(g, 32, 32, 4.0, 0.5, support=True)[0]) == [19, 17, 19, 63, 17, 45]
    assert list(O.rects(g, 32, 32, 4.0, 0.5)[0]) == [-22, -33, 0, 105, 0, 94]
    g["sigma"] = np.array([[2.0, 3.0]], np.float32)
    assert list(O.rects(g, 32, 32, 4.0, 0.1, support=True)[0]) == [29, 18, 29, 54, 18, 43]
    assert list(O.rects(g, 32, 32, 4.0, 0.1)[0]) == [29, 18, 29, 54, 18, 43]


@pytest.mark.parametrize("rho,sig", [(0.0, (0.3, 0.5)), (0.9, (0.4, 0.2)), (-0.99, (0.3, 0.3)),
                                     (0.5, (0.05, 0.7))])
def test_support_outside_below_fp32(rho, sig):
    """R21's premise, checked on the oracle's own fp64 Eq. 2: with the window covering the whole
    image (r = 1), every pixel outside the support rect receives < 2^-131 * alpha * c * K
    (K = 1/(2 pi sx sy sqrt(1 - rho^2)), the peak density), below fp32's smallest normal
    relative to the peak; the peak itself lies inside."""
    H, W, s = 8, 8, 4.0
    g = one(mu=(3.3, 4.1), sigma=sig, rho=rho)
    img = O.render_fwd(g, H, W, s, 1.0, mode="rect")[..., 0]
    _, _, x0, x1, y0, y1 = O.rects(g, H, W, s, 1.0, support=True)[0]
    K = 1.0 / (2 * math.pi * sig[0] * sig[1] * math.sqrt(1 - rho * rho))
    mask = np.ones_like(img, bool)
    mask[y0:y1 + 1, x0:x1 + 1] = False
    assert mask.any()
    assert img[mask].max() < 2.0 ** -131 * K
    assert img[~mask].max() == img.max() > 0


@pytest.mark.parametrize("cfg", [(10, 12, 4.0, 0.3, "image", 0), (9, 7, 2.5, 1.0, "stress", 1),
                                 (6, 11, 8.0, 0.5, "stress", 2), (12, 12, 1.0, 1.0, "image", 3),
                                 (7, 9, (6.0, 2.5), 0.5, "stress", 4)])
def test_support_render_equals_window_render(cfg):
    """R21: rendering over the support rects differs from the window sum of Alg. 1 only by terms
    below 2^-131 of each Gaussian's peak (forward and every gradient)."""
    H, W, s, r, dist, seed = cfg
    cl = S.gaussians(H, W, m=4, seed=seed, dist=dist, offset_range=1.5)
    a = O.render_fwd(cl, H, W, s, r, mode="rect")
    b = O.render_fwd(cl, H, W, s, r, mode="support")
    sx, sy = cl["sigma"][:, 0].astype(np.float64), cl["sigma"][:, 1].astype(np.float64)
    rh = cl["rho"].astype(np.float64)
    peak = np.abs(cl["alpha"]) * np.abs(cl["color"]).max(1) / (
        2 * np.pi * sx * sy * np.sqrt((1 - rh) * (1 + rh)))
    Hs, Ws = O.out_dims(H, W, s)
    bound = 2.0 ** -131 * float(peak.sum())
    assert np.abs(a - b).max() <= bound
    assert O.pair_count(cl, H, W, s, r, support=True) <= O.pair_count(cl, H, W, s, r)
    g = S.grad_out(a.shape, seed=seed)
    ga = O.render_bwd(cl, H, W, s, r, g, mode="rect")
    gb = O.render_bwd(cl, H, W, s, r, g, mode="support")
    for k in ga:
        # d/dtheta of a dropped term is (polynomial in Q <= 1e3 of it) x the term itself
        assert np.abs(ga[k] - gb[k]).max() <= 1e6 * bound * Hs * Ws / min(1.0, sx.min(),
                                                                          sy.min()) ** 2, k


# --------------------------------------------------------------------------- scale vector (R22)
@pytest.mark.parametrize("sw,sh,H,W", [(2, 3, 6, 7), (3, 2, 5, 4), (1, 4, 4, 6)])
def test_scale_vector_is_a_subsampling_of_the_isotropic_image(sw, sh, H, W):
    """R22 ("an upsampling scale vector"): with integer scales (sw, sh), pixel (x, y)
    samples (x/sw, y/sh) = (x k_x/L, y k_y/L) at the isotropic scale L = sw sh, i.e. pixel
    (sh x, sw y) of the isotropic image, with the same window test (r W, r H in LR units).
    The two quotients are correctly rounded from the same real, so in brute mode
    I_(sw,sh)[y, x] == I_L[sw y, sh x] bit for bit; a swapped axis or scale fails it."""
    r = 0.3
    L = float(sw * sh)
    cl = S.gaussians(H, W, m=4, seed=11, dist="stress", offset_range=1.5)
    a = O.render_fwd(cl, H, W, (float(sw), float(sh)), r, mode="brute")
    b = O.render_fwd(cl, H, W, L, r, mode="brute")
    assert a.shape[:2] == (sh * H, sw * W)
    assert np.array_equal(b[::sw, ::sh][:sh * H, :sw * W], a)
    assert a.any()


def test_scale_vector_transpose_symmetry():
    """Swapping the axes of the whole problem (mu, sigma, H <-> W, sw <-> sh; rho is symmetric in
    Eq. 2) transposes the rendered image and swaps the x/y gradients."""
    H, W, sw, sh, r = 5, 7, 2.5, 3.25, 0.3
    cl = {k: np.asarray(v, np.float64) for k, v in S.gaussians(H, W, m=4, seed=12).items()}
    tr = dict(cl, mu=cl["mu"][:, ::-1].copy(), sigma=cl["sigma"][:, ::-1].copy())
    a = O.render_fwd(cl, H, W, (sw, sh), r, mode="rect")
    b = O.render_fwd(tr, W, H, (sh, sw), r, mode="rect")
    assert a.shape[:2] == (int(math.floor(sh * H)), int(math.floor(sw * W)))
    np.testing.assert_allclose(b.transpose(1, 0, 2), a, rtol=1e-13, atol=1e-300)
    g = S.grad_out(a.shape, seed=5)
    ga = O.render_bwd(cl, H, W, (sw, sh), r, g, mode="rect")
    gb = O.render_bwd(tr, W, H, (sh, sw), r, g.transpose(1, 0, 2).copy(), mode="rect")
    for k in ("alpha", "rho", "color"):
        np.testing.assert_allclose(gb[k], ga[k], rtol=1e-11, atol=1e-14 * np.abs(ga[k]).max())
    for k in ("mu", "sigma"):
        np.testing.assert_allclose(gb[k][:, ::-1], ga[k], rtol=1e-11,
                                   atol=1e-14 * np.abs(ga[k]).max())


def test_scale_vector_single_gaussian_closed_form():
    """Eq. 2 at the R22 sample point: an axis-aligned Gaussian (rho = 0) centred at mu renders
    alpha c exp(-((x/sw - mu_x)^2/sx^2 + (y/sh - mu_y)^2/sy^2)/2) / (2 pi sx sy) at (x, y)."""
    sw, sh, mu, sig = 3.0, 1.5, (2.2, 3.1), (0.7, 1.3)
    a = O.render_fwd(one(mu=mu, sigma=sig, color=(1.0, 0.5, 2.0)), 6, 5, (sw, sh), 1.0,
                     mode="brute")
    for (x, y) in [(0, 0), (6, 4), (7, 5), (14, 8)]:
        X, Y = x / sw, y / sh
        want = math.exp(-0.5 * ((X - mu[0]) ** 2 / sig[0] ** 2 + (Y - mu[1]) ** 2 / sig[1] ** 2)) \
            / (2 * math.pi * sig[0] * sig[1])
        assert a[y, x, 0] == pytest.approx(want, rel=1e-13)
        assert a[y, x, 2] == pytest.approx(2 * want, rel=1e-13)


def test_scale_vector_window_per_axis():
    """R1/R2/R22: the window is |x/sw - mu_x| < r W and |y/sh - mu_y| < r H: with sw != sh the
    integer rect spans (about) 2 r W sw columns and 2 r H sh rows."""
    H, W, sw, sh, r = 10, 20, 2.0, 5.0, 0.1
    R = O.rects(one(mu=(10.0, 5.0)), H, W, (sw, sh), r)[0]
    # x: 10 +- 2 (LR) -> (16, 24) exclusive in HR px at sw = 2; y: 5 +- 1 -> (20, 30) at sh = 5
    assert list(R[2:]) == [17, 23, 21, 29]
