"""GPU parity: the sm_100a path (through the C-ABI) vs the float64 oracle, element by element on
the same seeded float32 inputs. Gates (reading R18): forward max-abs <= 1e-5 on the
image-like distribution (1e-5 * max(1,|I|) on the stress one); backward on image-like inputs
|g - g_ref| <= 1e-4 * max(|g_ref|, 1e-2 * S_t) with S_t the oracle's absolute term mass
(SURVEY 8(c).18), on the stress distribution R18's gate (tests/_util.gate_bounds); binning
bit-exact (rects, per-tile lists and their order)."""
import numpy as np
import pytest

import gsr_synth as S
import oracle as O
from _util import KEYS, assert_bwd_close, assert_fwd_close, cat, grad_dict, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gsr():
    import torch
    import paper_2501_06838_b200 as g
    from paper_2501_06838_b200.build import build
    assert torch.cuda.is_available()
    build()
    g.load()
    return g


def fwd(gsr, cloud, H, W, s, r=0.1):
    import torch
    out = gsr.render_fwd(*to_dev(cloud), H, W, s, ratio=r)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def bwd(gsr, cloud, H, W, s, g, r=0.1):
    import torch
    grads = gsr.render_bwd(*to_dev(cloud), H, W, s, torch.from_numpy(g).cuda(), ratio=r)
    torch.cuda.synchronize()
    return grad_dict(grads)


# --------------------------------------------------------------------------- binning, bit-exact
def adversarial_cloud(H, W, s, seed=0):
    """Image-like cloud plus centres placed on tile edges, on exact window-edge values, outside
    the image, huge, and invalid parameters."""
    c = S.gaussians(H, W, m=4, seed=seed, offset_range=1.0)
    n = c["alpha"].shape[0]
    rng = np.random.default_rng(seed + 1)
    k = min(n, 64)
    idx = rng.choice(n, k, replace=False)
    mu = c["mu"].copy()
    tw = 32.0 / s
    mu[idx[:8], 0] = np.float32(tw * rng.integers(0, 4, 8))            # on tile edges (LR px)
    mu[idx[8:16], 1] = np.float32(tw * rng.integers(0, 4, 8))
    mu[idx[16:24], 0] = np.float32(0.1 * W + rng.integers(0, 3, 8) / s)  # window edge on a pixel
    mu[idx[24:28]] = np.float32([[-0.3 * W, 2], [W + 0.05 * W, 1], [2, -0.25 * H], [1, H * 1.2]])
    mu[idx[28:30]] = np.float32([[1e9, 3], [-3e30, 2]])                   # huge
    c["mu"] = mu
    c["sigma"][idx[30], 0] = 0.0                                          # invalid
    c["rho"][idx[31]] = np.float32(1.0)
    c["alpha"][idx[32]] = np.float32(np.nan)
    c["color"][idx[33], 1] = np.float32(np.inf)
    return c


@pytest.mark.parametrize("support", [False, True])
@pytest.mark.parametrize("H,W,s,r", [(48, 48, 4.0, 0.1), (20, 33, 2.7, 0.1), (9, 13, 30.0, 0.1),
                                     (16, 16, 1.0, 0.5), (12, 10, 3.3, 1.0)])
def test_rects_bit_exact(gsr, H, W, s, r, support):
    """Window rects (R2) and support rects (R21) as the GPU computes them == the oracle's."""
    import paper_2501_06838_b200.debug as D
    c = adversarial_cloud(H, W, s)
    got = D.rects(*to_dev(c), H, W, s, r, support=support).cpu().numpy()
    ref = O.rects(c, H, W, s, r, support=support)
    empty_ref = (ref[:, 2] > ref[:, 3]) | (ref[:, 4] > ref[:, 5])
    empty_got = (got[:, 0] > got[:, 1]) | (got[:, 2] > got[:, 3])
    assert np.array_equal(empty_ref, empty_got)
    ne = ~empty_ref
    assert np.array_equal(got[ne], ref[ne][:, 2:6].astype(np.int32))


@pytest.mark.parametrize("H,W,s,r", [(48, 48, 4.0, 0.1), (20, 33, 2.7, 0.1), (9, 13, 30.0, 0.1),
                                     (12, 10, 3.3, 1.0)])
def test_tile_lists_bit_exact(gsr, H, W, s, r):
    """Per-tile Gaussian lists the render kernels visit (support rects, R21) == CPU brute force
    (O(N*tiles)), and their order is (cell, index) ascending -- the stable sort."""
    import paper_2501_06838_b200.debug as D
    c = adversarial_cloud(H, W, s, seed=3)
    tw, th, cw, ch = gsr.tile_shape()
    counts, ids, cells = [t.cpu().numpy() for t in D.tile_lists(*to_dev(c), H, W, s, r)]
    rc, rids = O.tile_lists(c, H, W, s, r, tw, th, support=True)
    assert np.array_equal(counts.astype(np.int64), rc)
    off = np.concatenate([[0], np.cumsum(counts)])
    for t in range(len(counts)):
        a = ids[off[t]:off[t + 1]].astype(np.int64)
        b = rids[off[t]:off[t + 1]]
        assert np.array_equal(np.sort(a), b), t
        key = cells[off[t]:off[t + 1]].astype(np.int64) * (1 << 32) + a
        assert np.all(np.diff(key) > 0), t


def test_pair_count(gsr):
    import torch
    for (H, W, s) in [(48, 48, 4.0), (9, 13, 30.0), (20, 33, 2.7)]:
        c = adversarial_cloud(H, W, s)
        lay = gsr.layout([gsr.Image(H, W, s, 0, c["alpha"].shape[0])])
        assert gsr.pair_count(*to_dev(c), lay) == O.pair_count(c, H, W, s)
        assert (gsr.pair_count(*to_dev(c), lay, support=True) ==
                O.pair_count(c, H, W, s, support=True))


# --------------------------------------------------------------------------- forward
@pytest.mark.parametrize("dist", ["image", "stress"])
def test_fwd_c1(gsr, dist):
    """C1: 48x48 LR patch at x4 -> 192x192, full image vs oracle."""
    H, W, s = 48, 48, 4.0
    c = S.gaussians(H, W, seed=1001, dist=dist)
    got = fwd(gsr, c, H, W, s)
    want = O.render_fwd(c, H, W, s, 0.1, mode="rect")
    assert got.shape == want.shape == (192, 192, 3)
    assert_fwd_close(got, want, dist)


@pytest.mark.parametrize("H,W,s,r", [(1, 1, 1.0, 0.1), (3, 5, 1.0, 1.0), (7, 9, 2.5, 0.1),
                                     (13, 11, 3.7, 0.3), (5, 40, 6.1, 0.1), (33, 17, 1.9, 0.1),
                                     (6, 6, 17.0, 0.1), (10, 12, 4.0, 1.0)])
def test_fwd_ragged_shapes(gsr, H, W, s, r):
    """Non-multiple-of-tile sizes, s = 1, non-integer s, r = 1 (window = whole image)."""
    c = S.gaussians(H, W, seed=int(100 * s) + H, offset_range=1.0)
    assert_fwd_close(fwd(gsr, c, H, W, s, r), O.render_fwd(c, H, W, s, r))


@pytest.mark.parametrize("s,r,sig,dist", [(2.0, 0.6, 1.0, "image"), (3.0, 0.4, 1.0, "image"),
                                          (4.0, 0.3, 1.0, "image"), (8.0, 0.3, 1.0, "image"),
                                          (4.0, 0.3, 0.5, "image"), (4.0, 0.3, 2.0, "image"),
                                          (3.0, 0.4, 1.0, "stress"), (2.5, 0.5, 0.7, "stress")])
def test_fwd_recurrence_regime(gsr, s, r, sig, dist):
    """Windows >= 48 HR px (2-row lane blocks) with D = a1/s spanning both sides of the
    exponential-recurrence threshold (render_fwd.cu, MODE 2: D <= 1), full image vs oracle."""
    H, W = 24, 24
    c = S.gaussians(H, W, m=4, seed=int(10 * s) + int(10 * sig), dist=dist)
    c["sigma"] = (c["sigma"] * np.float32(sig)).astype(np.float32)
    assert_fwd_close(fwd(gsr, c, H, W, s, r), O.render_fwd(c, H, W, s, r, mode="rect"), dist)


def test_fwd_adversarial_and_empty(gsr):
    H, W, s = 20, 33, 2.7
    c = adversarial_cloud(H, W, s)
    assert_fwd_close(fwd(gsr, c, H, W, s), O.render_fwd(c, H, W, s, 0.1))
    e = {k: v[:0] for k, v in c.items()}
    import torch
    out = gsr.render_fwd(*[torch.zeros((0,) + v.shape[1:], device="cuda") for v in e.values()],
                         H, W, s)
    assert out.shape == (54, 89, 3) and not out.abs().sum().item()


@pytest.mark.parametrize("H,W,s", [(30, 30, 3.0), (60, 80, 8.0), (170, 255, 8.0)],
                         ids=["small-tiles", "large-tiles-split-k", "c5-image"])
def test_fwd_deterministic(gsr, H, W, s):
    """Bitwise run-to-run reproducibility: the candidate stream's lane interleave assigns every
    candidate to a fixed warp (and split-K cluster CTA), and the warp images are summed in a
    fixed order -- small tiles, large tiles under split-K, and a C5 image (cell-reach trim)."""
    c = S.gaussians(H, W, seed=5)
    a = fwd(gsr, c, H, W, s)
    b = fwd(gsr, c, H, W, s)
    assert np.array_equal(a, b)


def test_fwd_c4_rows(gsr):
    """C4: 68x45 at x30 -> 2040x1350 (window 408x270 px); rows sampled incl. edges."""
    H, W, s = 45, 68, 30.0
    c = S.gaussians(H, W, seed=1004)
    got = fwd(gsr, c, H, W, s)
    for rows in [(0, 3), (517, 520), (1347, 1350)]:
        want = O.render_fwd(c, H, W, s, 0.1, rows=rows)
        assert_fwd_close(got[rows[0]:rows[1]], want)


def test_fwd_stream_chunks_and_reach(gsr):
    """A dense image (64 Gaussians per cell) with very wide supports (every 50th Gaussian at
    sigma = 3 LR px, r = 1): the forward's candidate stream spans > 32 cell rows per tile
    (several chunks, rebuilt under the CTA barriers) and trims them by the cell reach."""
    H, W, s = 40, 60, 8.0
    c = S.gaussians(H, W, seed=1005)
    c["sigma"][::50] = 3.0
    got = fwd(gsr, c, H, W, s, r=1.0)
    for rows in [(0, 3), (150, 153), (317, 320)]:
        want = O.render_fwd(c, H, W, s, 1.0, rows=rows)
        assert_fwd_close(got[rows[0]:rows[1]], want)


def test_fwd_c3_pixels(gsr):
    """C3: 510x339 at x4 -> 2040x1356, N = 2.77M; sampled pixels vs the brute-force oracle."""
    H, W, s = 339, 510, 4.0
    c = S.gaussians(H, W, seed=1003)
    got = fwd(gsr, c, H, W, s)
    assert got.shape == (1356, 2040, 3)
    rng = np.random.default_rng(0)
    px = np.concatenate([rng.integers(0, 2040, 40), [0, 2039, 0, 2039, 1023]])
    py = np.concatenate([rng.integers(0, 1356, 40), [0, 0, 1355, 1355, 677]])
    want = O.render_pixels(c, H, W, s, 0.1, px, py)
    assert_fwd_close(got[py, px], want)


def test_fwd_c3_full_row_band(gsr):
    """C3: one full 16-row band (all 2040 columns, rows 664..679 cross the forward-tile and cell
    row seam at 672) vs the full-window oracle (rect mode)."""
    H, W, s = 339, 510, 4.0
    c = S.gaussians(H, W, seed=1003)
    got = fwd(gsr, c, H, W, s)
    want = O.render_fwd(c, H, W, s, 0.1, mode="rect", rows=(664, 680))
    assert_fwd_close(got[664:680], want)


# --------------------------------------------------------------------------- backward
@pytest.mark.parametrize("dist", ["image", "stress"])
def test_bwd_c1(gsr, dist):
    H, W, s = 48, 48, 4.0
    c = S.gaussians(H, W, seed=1001, dist=dist)
    g = S.grad_out((192, 192, 3), seed=2001)
    got = bwd(gsr, c, H, W, s, g)
    want = O.render_bwd(c, H, W, s, 0.1, g, want_absmass=True)
    stats = assert_bwd_close(got, want, want["absmass"], dist=dist)
    print("C1 bwd rel-err p50/p99, worst bound ratio:", stats)


@pytest.mark.parametrize("H,W,s,r", [(1, 1, 1.0, 0.1), (7, 9, 2.5, 0.1), (13, 11, 3.7, 0.3),
                                     (5, 40, 6.1, 0.1), (6, 6, 17.0, 0.1), (10, 12, 4.0, 1.0)])
def test_bwd_ragged_shapes(gsr, H, W, s, r):
    c = S.gaussians(H, W, seed=int(10 * s) + W, offset_range=1.0)
    Hs, Ws = O.out_dims(H, W, s)
    g = S.grad_out((Hs, Ws, 3), seed=7)
    got = bwd(gsr, c, H, W, s, g, r)
    want = O.render_bwd(c, H, W, s, r, g, want_absmass=True)
    assert_bwd_close(got, want, want["absmass"])


def test_bwd_adversarial_invalid_zero(gsr):
    H, W, s = 20, 33, 2.7
    c = adversarial_cloud(H, W, s)
    Hs, Ws = O.out_dims(H, W, s)
    g = S.grad_out((Hs, Ws, 3), seed=8)
    got = bwd(gsr, c, H, W, s, g)
    want = O.render_bwd(c, H, W, s, 0.1, g, want_absmass=True)
    assert_bwd_close(got, want, want["absmass"])
    R = O.rects(c, H, W, s, 0.1)
    dead = (R[:, 2] > R[:, 3]) | (R[:, 4] > R[:, 5])
    for k in KEYS:
        assert not np.any(got[k][dead]), k       # pruning consistency: exactly zero


def test_bwd_c4_sampled(gsr):
    """C4 (wide footprints): gradients of a sample of Gaussians vs the oracle (idx mode)."""
    H, W, s = 45, 68, 30.0
    c = S.gaussians(H, W, seed=1004)
    g = S.grad_out((1350, 2040, 3), seed=2004)
    got = bwd(gsr, c, H, W, s, g)
    rng = np.random.default_rng(1)
    idx = np.concatenate([rng.choice(c["alpha"].shape[0], 60, replace=False), [0, 48959]])
    want = O.render_bwd(c, H, W, s, 0.1, g, idx=idx, want_absmass=True)
    assert_bwd_close({k: got[k][idx] for k in KEYS}, want, want["absmass"])


# --------------------------------------------------------------------------- batched / ragged
def test_c2_batch_fwd_bwd(gsr):
    """C2: 16 patches of 48x48 with s ~ U[1,4] (seed 0), one batched call each way."""
    import torch
    imgs = [(48, 48, float(s)) for s in S.c2_scales()]
    clouds = [S.gaussians(48, 48, seed=1002 + 17 * k) for k in range(16)]
    allc = cat(clouds)
    counts = [cl["alpha"].shape[0] for cl in clouds]
    dev = to_dev(allc)
    for t in dev:
        t.requires_grad_(True)
    flat, lay = gsr.render_batch(*dev, imgs, counts)
    gflat = torch.from_numpy(S.grad_out((lay.out_numel,), seed=2002)).cuda()
    (flat * gflat).sum().backward()
    torch.cuda.synchronize()
    gnp = gflat.cpu().numpy()
    grads = grad_dict([t.grad for t in dev])
    off = 0
    for k, ((H, W, s), cl) in enumerate(zip(imgs, clouds)):
        want = O.render_fwd(cl, H, W, s, 0.1)
        got = lay.view(flat.detach(), k).cpu().numpy()
        assert_fwd_close(got, want)
        gk = lay.view(torch.from_numpy(gnp), k).numpy()
        wb = O.render_bwd(cl, H, W, s, 0.1, gk, want_absmass=True)
        n = cl["alpha"].shape[0]
        assert_bwd_close({kk: grads[kk][off:off + n] for kk in KEYS}, wb, wb["absmass"])
        off += n


def test_batch_image_order_invariance(gsr):
    """The render kernels launch the images' tiles densest-first (ImgTable::sched); every tile is
    computed from its own image's Gaussians only, so permuting the images of a ragged batch gives
    each image the same bits (forward) and the same gradients up to the fp64 atomics' order."""
    import torch
    imgs = [(48, 48, float(s)) for s in S.c2_scales()][:8]
    clouds = [S.gaussians(48, 48, seed=3100 + k) for k in range(8)]
    grads_img = [S.grad_out(tuple(O.out_dims(H, W, s)) + (3,), seed=3200 + k)
                 for k, (H, W, s) in enumerate(imgs)]

    def run(order):
        cl = [clouds[k] for k in order]
        dev = to_dev(cat(cl))
        ims, off = [], 0
        for k in order:
            H, W, s = imgs[k]
            n = clouds[k]["alpha"].shape[0]
            ims.append(gsr.Image(H, W, s, off, n))
            off += n
        lay = gsr.layout(ims)
        out = gsr.render_fwd_batched(*dev, lay)
        g = torch.cat([torch.from_numpy(grads_img[k].reshape(-1)) for k in order]).cuda()
        grads = gsr.render_bwd_batched(*dev, lay, g)
        torch.cuda.synchronize()
        res, goff = {}, 0
        for j, k in enumerate(order):
            n = clouds[k]["alpha"].shape[0]
            res[k] = (lay.view(out, j).cpu().numpy(),
                      [t[goff:goff + n].cpu().numpy() for t in grads])
            goff += n
        return res

    a = run(list(range(8)))
    b = run(list(range(7, -1, -1)))
    for k in range(8):
        assert np.array_equal(a[k][0], b[k][0])
        for ga, gb in zip(a[k][1], b[k][1]):
            np.testing.assert_allclose(ga, gb, rtol=1e-6, atol=1e-12 * max(1.0, np.abs(ga).max()))


def test_row_bands_equal_full(gsr):
    """Row-band rendering (the multi-GPU shard) reproduces the rows of the full render, and band
    moments sum to the full moments."""
    import torch
    H, W, s = 24, 30, 3.0
    c = S.gaussians(H, W, seed=9)
    n = c["alpha"].shape[0]
    dev = to_dev(c)
    full = gsr.render_fwd(*dev, H, W, s)
    Hs, Ws = full.shape[:2]
    bands = [(0, 20), (20, 45), (45, Hs)]
    g = torch.from_numpy(S.grad_out((Hs, Ws, 3), seed=3)).cuda()
    mom = torch.zeros((n, 8), dtype=torch.float64, device="cuda")
    for rb, re in bands:
        lay = gsr.layout([gsr.Image(H, W, s, 0, n, rb, re)])
        part = gsr.render_fwd_batched(*dev, lay)
        assert torch.allclose(part.view(re - rb, Ws, 3), full[rb:re], rtol=1e-6, atol=1e-7)
        gsr.render_bwd_moments_batched(*dev, lay, g[rb:re].reshape(-1).contiguous(), mom)
    grads_b = gsr.finalize_grads(*dev, mom)
    grads_f = gsr.render_bwd(*dev, H, W, s, g)
    for a, b in zip(grads_b, grads_f):       # same sums, different fp32 grouping
        assert torch.allclose(a, b, rtol=1e-4, atol=1e-6 * b.abs().max().item())


def test_autograd_matches_abi(gsr):
    import torch
    H, W, s = 16, 16, 2.0
    c = S.gaussians(H, W, seed=4)
    dev = to_dev(c)
    for t in dev:
        t.requires_grad_(True)
    img = gsr.render(*dev, H, W, s)
    g = torch.from_numpy(S.grad_out(tuple(img.shape), seed=5)).cuda()
    grads = torch.autograd.grad(img, dev, g)
    ref = gsr.render_bwd(*[t.detach() for t in dev], H, W, s, g)
    for a, b in zip(grads, ref):
        assert torch.equal(a, b) or torch.allclose(a, b, rtol=1e-6, atol=1e-9)


def test_cpu_tensors_rejected(gsr):
    import torch
    c = S.gaussians(4, 4, seed=0)
    with pytest.raises(TypeError):
        gsr.render_fwd(*[torch.from_numpy(c[k]) for k in KEYS], 4, 4, 2.0)


@pytest.mark.parametrize("m,r", [(1, 0.01), (9, 0.01), (9, 0.4), (4, 0.8)])
def test_sweep_densities_and_ratios(gsr, m, r):
    """NEXT-3 sweep settings (m in {1,4,9}, r in {0.01 .. 0.8}) at a small size: fwd + bwd."""
    H, W, s = 18, 20, 4.0
    c = S.gaussians(H, W, m=m, seed=m * 10 + int(100 * r))
    Hs, Ws = O.out_dims(H, W, s)
    assert_fwd_close(fwd(gsr, c, H, W, s, r), O.render_fwd(c, H, W, s, r))
    g = S.grad_out((Hs, Ws, 3), seed=m)
    got = bwd(gsr, c, H, W, s, g, r)
    want = O.render_bwd(c, H, W, s, r, g, want_absmass=True)
    assert_bwd_close(got, want, want["absmass"])


def test_reuse_binning_matches_rebinning(gsr):
    """GSR_REUSE_BINNING (the forward's workspace) gives exactly the re-binned backward."""
    import torch
    H, W, s = 20, 18, 3.0
    c = S.gaussians(H, W, seed=21)
    dev = to_dev(c)
    lay = gsr.layout([gsr.Image(H, W, s, 0, c["alpha"].shape[0])])
    from paper_2501_06838_b200 import ops
    ws = ops.workspace_for(dev[0], lay)
    out = gsr.render_fwd_batched(*dev, lay, workspace=ws)
    g = torch.from_numpy(S.grad_out((lay.out_numel,), seed=2)).cuda()
    a = gsr.render_bwd_batched(*dev, lay, g, workspace=ws, reuse_binning=True)
    b = gsr.render_bwd_batched(*dev, lay, g)
    torch.cuda.synchronize()
    for x, y in zip(a, b):
        assert torch.allclose(x, y, rtol=1e-6, atol=1e-9)


def test_validate_params(gsr):
    """gsr_validate_params reports exactly the Gaussians outside the domain (R20)."""
    c = adversarial_cloud(20, 33, 2.7)
    a = np.concatenate([c[k].reshape(len(c["alpha"]), -1) for k in KEYS], 1)
    bad = ~np.isfinite(a).all(1) | (c["sigma"][:, 0] <= 0) | (c["sigma"][:, 1] <= 0) | \
        (np.abs(c["rho"]) >= 1)
    cnt, first = gsr.validate_params(*to_dev(c))
    assert cnt == int(bad.sum()) > 0 and first == int(np.nonzero(bad)[0][0])
    ok = S.gaussians(10, 10, seed=1)
    assert gsr.validate_params(*to_dev(ok)) == (0, -1)


def test_debug_validation_and_nvtx_env(tmp_path):
    """GSR_DEBUG=1: a render call on parameters outside the domain raises before any kernel runs
    (SURVEY §5); GSR_NVTX=1: the NVTX phase ranges leave the results unchanged."""
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    code = """
import sys, numpy as np, torch
sys.path.insert(0, %r)
import gsr_synth as S, paper_2501_06838_b200 as gsr
c = S.gaussians(12, 14, seed=3)
dev = [torch.from_numpy(c[k]).cuda() for k in ("alpha", "mu", "sigma", "rho", "color")]
ok = gsr.render(*dev, 12, 14, 3.0)
dev[2][5, 1] = -1.0
try:
    gsr.render(*dev, 12, 14, 3.0)
    print("NO-RAISE")
except ValueError as e:
    print("RAISED", "first index 5" in str(e))
np.save(sys.argv[1], ok.cpu().numpy())
""" % str(root)
    outs = {}
    for env in ({"GSR_DEBUG": "1"}, {"GSR_DEBUG": "1", "GSR_NVTX": "1"}):
        f = tmp_path / ("nvtx.npy" if "GSR_NVTX" in env else "plain.npy")
        r = subprocess.run([sys.executable, "-c", code, str(f)], capture_output=True, text=True,
                           env={**__import__("os").environ, **env}, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        assert "RAISED True" in r.stdout, r.stdout
        outs[f.name] = np.load(f)
    assert np.array_equal(outs["plain.npy"], outs["nvtx.npy"])


def _tile_pairs(rects, Hs, Ws, tw, th):
    """Brute force: sorted (tile, gaussian) keys of every support rect x forward tile overlap."""
    x0, x1, y0, y1 = (rects[:, k].astype(np.int64) for k in range(4))
    ok = (x0 <= x1) & (y0 <= y1)
    ntx = -(-Ws // tw)
    keys = []
    for i in np.nonzero(ok)[0]:
        txs = np.arange(x0[i] // tw, x1[i] // tw + 1)
        tys = np.arange(y0[i] // th, y1[i] // th + 1)
        t = (tys[:, None] * ntx + txs[None, :]).ravel()
        keys.append(t * (1 << 32) + i)
    return np.sort(np.concatenate(keys)) if keys else np.zeros(0, np.int64)


@pytest.mark.parametrize("H,W,s,r,wide", [(48, 48, 4.0, 0.1, False), (60, 80, 8.0, 0.1, False),
                                          (40, 60, 8.0, 1.0, True)],
                         ids=["small-tiles", "large-tiles-reach-trim", "multi-chunk"])
def test_fwd_tile_lists_bit_exact(gsr, H, W, s, r, wide):
    """K4's kept candidates per forward tile (its candidate stream -- cell rows trimmed by the
    cell reach -- and filter, materialised through gsr_debug_fwd_tile_lists) equal the brute-force
    set of support rects (R21) meeting the tile, without duplicates; every path is consistent
    with the rects: a single column half only when the support misses the other, the full-window
    paths only where the window covers the tile (large) / cuts no support edge inside it (small)."""
    import torch
    from paper_2501_06838_b200 import debug
    c = S.gaussians(H, W, seed=1007)
    if wide:
        c["sigma"][::50] = 3.0
    dev = to_dev(c)
    (tw, th, nt), counts, ids, paths = debug.fwd_tile_lists(*dev, H, W, s, r)
    sup = debug.rects(*dev, H, W, s, r, support=True).cpu().numpy()
    win = debug.rects(*dev, H, W, s, r).cpu().numpy()
    Hs, Ws = O.out_dims(H, W, s)
    assert (tw, th) in ((16, 8), (32, 16))
    counts, ids, paths = counts.cpu().numpy(), ids.cpu().numpy(), paths.cpu().numpy()
    tiles = np.repeat(np.arange(nt), counts)
    got = tiles.astype(np.int64) * (1 << 32) + ids
    assert len(np.unique(got)) == len(got), "a candidate kept twice in one tile"
    assert np.array_equal(np.sort(got), _tile_pairs(sup, Hs, Ws, tw, th))
    ntx = -(-Ws // tw)
    tx0 = (tiles % ntx) * tw
    ty0 = (tiles // ntx) * th
    sx0, sx1, wx0, wx1 = sup[ids, 0], sup[ids, 1], win[ids, 0], win[ids, 1]
    sy0, sy1, wy0, wy1 = sup[ids, 2], sup[ids, 3], win[ids, 2], win[ids, 3]
    if tw == 32:
        hv = paths % 3
        assert np.all(sx1[hv == 1] <= tx0[hv == 1] + 15)
        assert np.all(sx0[hv == 2] >= tx0[hv == 2] + 16)
        both = hv == 0
        assert np.all((sx0[both] <= tx0[both] + 15) & (sx1[both] >= tx0[both] + 16))
        covers = (wx0 <= tx0) & (wx1 >= np.minimum(tx0 + tw - 1, Ws - 1)) & (wy0 <= ty0) & \
                 (wy1 >= ty0 + th - 1)
        assert np.array_equal(paths < 6, covers)       # recurrence / direct only when covered
    else:
        fx1 = np.minimum(tx0 + tw - 1, Ws - 1)
        cut = ((wx0 > tx0) & (sx0 == wx0)) | ((wx1 < fx1) & (sx1 == wx1)) | \
              ((wy0 > ty0) & (sy0 == wy0)) | ((wy1 < ty0 + th - 1) & (sy1 == wy1))
        assert np.array_equal(paths >= 3, cut)


def test_fwd_output_at_any_float_offset(gsr):
    """The caller's output buffer need not be 16-B aligned (a view one float into a tensor): the
    epilogue's float4 row stores fall back to scalar stores where the row is misaligned, and the
    image is bit-identical to the aligned render (large and small tiles)."""
    import torch
    for H, W, s in [(21, 30, 8.0), (15, 19, 2.5)]:
        c = S.gaussians(H, W, seed=9)
        dev = to_dev(c)
        lay = gsr.layout([gsr.Image(H, W, s, 0, c["alpha"].shape[0])])
        ref = gsr.render_fwd_batched(*dev, lay)
        for shift in (1, 2, 3):
            buf = torch.full((lay.out_numel + 4,), float("nan"), device="cuda")
            out = buf[shift:shift + lay.out_numel]
            gsr.render_fwd_batched(*dev, lay, out=out)
            torch.cuda.synchronize()
            assert torch.equal(out, ref)
