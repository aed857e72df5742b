"""GPU parity at BASELINE.json's full C5 size, in the launch configuration bench.py times: 64
DIV2K-size images (255x170 LR at x8 -> 2040x1360) in one batched call with a private
workspace, the forward's binning reused by the backward moments (GSR_REUSE_BINNING), then the
finalize -- checked on sampled outputs the float64 oracle computes one by one: pixels of three
images (random + corners), and the gradients of sampled Gaussians (oracle idx mode)."""
import numpy as np
import pytest

import gsr_synth as S
import oracle as O
from _util import KEYS, assert_bwd_close, assert_fwd_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c5():
    """The whole C5 step on the GPU in bench.py's launch configuration (computed once)."""
    import torch
    import paper_2501_06838_b200 as gsr
    from paper_2501_06838_b200 import ops
    imgs = S.CONFIGS["C5"]["images"]
    assert len(imgs) == 64
    clouds = [S.gaussians(H, W, seed=1000 + k) for k, (H, W, s) in enumerate(imgs)]
    counts = [c["alpha"].shape[0] for c in clouds]
    offs = np.concatenate([[0], np.cumsum(counts)])
    dev = [torch.from_numpy(np.concatenate([c[k] for c in clouds])).cuda() for k in KEYS]
    lay = gsr.layout([gsr.Image(H, W, s, int(offs[k]), counts[k])
                      for k, (H, W, s) in enumerate(imgs)])
    g = torch.empty(lay.out_numel, dtype=torch.float32, device="cuda")
    g.uniform_(-1.0, 1.0, generator=torch.Generator(device="cuda").manual_seed(2000))
    ws = ops.workspace_for(dev[0], lay, 0.1)
    out = gsr.render_fwd_batched(*dev, lay, 0.1, workspace=ws)
    mom = torch.zeros((dev[0].shape[0], 8), dtype=torch.float64, device="cuda")
    gsr.render_bwd_moments_batched(*dev, lay, g, mom, 0.1, workspace=ws, reuse_binning=True)
    grads = dict(zip(KEYS, gsr.finalize_grads(*dev, mom)))
    torch.cuda.synchronize()
    del mom, ws
    return dict(imgs=imgs, clouds=clouds, counts=counts, offs=offs, lay=lay, out=out, g=g,
                grads=grads)


def test_c5_full_size_sampled(c5):
    import torch
    imgs, clouds, counts, offs, lay = c5["imgs"], c5["clouds"], c5["counts"], c5["offs"], c5["lay"]
    out, g, grads = c5["out"], c5["g"], c5["grads"]
    rng = np.random.default_rng(5)
    H, W, s = imgs[0]
    Hs, Ws = O.out_dims(H, W, s)
    for k in (0, 31, 63):
        img = lay.view(out, k).cpu().numpy()
        px = np.concatenate([rng.integers(0, Ws, 24), [0, Ws - 1, 0, Ws - 1]])
        py = np.concatenate([rng.integers(0, Hs, 24), [0, 0, Hs - 1, Hs - 1]])
        assert_fwd_close(img[py, px], O.render_pixels(clouds[k], H, W, s, 0.1, px, py))
    for k in (0, 63):
        gk = lay.view(g, k).cpu().numpy()
        idx = np.concatenate([rng.choice(counts[k], 14, replace=False), [0, counts[k] - 1]])
        want = O.render_bwd(clouds[k], H, W, s, 0.1, gk, idx=idx, want_absmass=True)
        sel = torch.from_numpy(offs[k] + idx).cuda()
        got = {kk: grads[kk][sel].cpu().numpy().astype(np.float64) for kk in KEYS}
        assert_bwd_close(got, want, want["absmass"])


@pytest.mark.parametrize("k,rows", [(0, (504, 520)), (37, (1000, 1016))])
def test_c5_full_row_bands(c5, k, rows):
    """Two full 16-row bands (all 2040 columns) of C5 images, each crossing a forward-tile row
    seam (multiples of 16 HR rows), backward-tile seams (8 rows) and a binning-cell row seam,
    vs the full-window oracle (rect mode, Alg. 1, Eq. 4)."""
    H, W, s = c5["imgs"][k]
    img = c5["lay"].view(c5["out"], k).cpu().numpy()
    want = O.render_fwd(c5["clouds"][k], H, W, s, 0.1, mode="rect", rows=rows)
    assert want.shape == (16, 2040, 3)
    assert_fwd_close(img[rows[0]:rows[1]], want)


def test_c5_gradients_1000_gaussians(c5):
    """Gradients of >= 1000 Gaussians of one C5 image vs the oracle: random ones, Gaussians whose
    support rect (R21) straddles a forward column-half seam (x = 16 mod 32) or a tile / cell
    seam (x = 0 mod 32), and Gaussians clipped by the image border."""
    import torch
    k = 11
    H, W, s = c5["imgs"][k]
    cl = c5["clouds"][k]
    n = c5["counts"][k]
    R = O.rects(cl, H, W, s, 0.1, support=True)
    x0, x1, y0, y1 = R[:, 2], R[:, 3], R[:, 4], R[:, 5]
    ok = (x0 <= x1) & (y0 <= y1)
    half = ok & ((x0 // 16) != (x1 // 16)) & ((x1 - x0) < 16 + 32)
    half &= ((x0 // 32) == (x1 // 32))                 # inside one 32-col tile, both halves
    seam = ok & ((x0 // 32) != (x1 // 32))
    Hs, Ws = O.out_dims(H, W, s)
    edge = ok & ((x0 == 0) | (x1 == Ws - 1) | (y0 == 0) | (y1 == Hs - 1))
    rng = np.random.default_rng(12)
    pick = lambda m, c: rng.choice(np.nonzero(m)[0], min(c, int(m.sum())), replace=False)
    idx = np.unique(np.concatenate([rng.choice(n, 400, replace=False), pick(half, 250),
                                    pick(seam, 250), pick(edge, 200), [0, n - 1]]))
    assert idx.size >= 1000 and half[idx].sum() >= 100
    gk = c5["lay"].view(c5["g"], k).cpu().numpy()
    want = O.render_bwd(cl, H, W, s, 0.1, gk, idx=idx, want_absmass=True)
    sel = torch.from_numpy(c5["offs"][k] + idx).cuda()
    got = {kk: c5["grads"][kk][sel].cpu().numpy().astype(np.float64) for kk in KEYS}
    assert_bwd_close(got, want, want["absmass"])


def test_band_partials_and_seam_set():
    """The row-band exchange of dist.py on the CUDA path, emulated in one process (this run has
    one GPU): G = 4 pair-balanced bands of a C5-geometry image; each band's moments are
    finalized on their own (the finalize is linear in the moments); bands and seam set from
    libgsr's K7 planner on the device; a Gaussian outside the seam
    set has a nonzero partial in at most one band, where it equals the oracle's gradient; the
    band partials summed over the seam set equal the whole-image gradients."""
    import torch
    import paper_2501_06838_b200 as gsr
    from paper_2501_06838_b200 import dist as gd
    H, W, s, G = 60, 90, 8.0, 4
    c = S.gaussians(H, W, seed=77)
    n = c["alpha"].shape[0]
    dev = [torch.from_numpy(c[k]).cuda() for k in KEYS]
    whole = [(H, W, s, 0, n)]
    rc = gd.row_pair_counts(dev, whole, 0.1)[0]
    b = gd.plan_bands(rc, G)
    seam = gd.seam_mask(gd.band_spans(dev, whole, [b], 0.1)).cpu().numpy()
    assert 0 < seam.sum() < n
    Hs, Ws = O.out_dims(H, W, s)
    g = torch.from_numpy(S.grad_out((Hs, Ws, 3), seed=78)).cuda()
    parts = []
    for r in range(G):
        lay = gsr.layout([gsr.Image(H, W, s, 0, n, b[r], b[r + 1])])
        mom = torch.zeros((n, 8), dtype=torch.float64, device="cuda")
        gsr.render_bwd_moments_batched(*dev, lay, g[b[r]:b[r + 1]].reshape(-1).contiguous(),
                                       mom, 0.1)
        gr = gsr.finalize_grads(*dev, mom)
        parts.append(np.concatenate([t.view(n, -1).cpu().numpy() for t in gr], 1)
                     .astype(np.float64))
    P = np.stack(parts)                                     # [G, n, 9]
    nz = (P != 0).any(2).sum(0)                             # bands with a nonzero partial
    assert (nz[~seam] <= 1).all()
    full_lay = gsr.layout([gsr.Image(H, W, s, 0, n)])
    full = np.concatenate([t.view(n, -1).cpu().numpy() for t in
                           gsr.render_bwd_batched(*dev, full_lay, g.reshape(-1), 0.1)], 1)
    tot = P.sum(0)
    scale = np.abs(full).max(0, keepdims=True)
    assert (np.abs(tot - full) <= 1e-5 * scale).all()
    rng = np.random.default_rng(3)
    idx = np.concatenate([rng.choice(np.nonzero(~seam)[0], 12, replace=False),
                          rng.choice(np.nonzero(seam)[0], 12, replace=False)])
    want = O.render_bwd(c, H, W, s, 0.1, g.cpu().numpy(), idx=idx, want_absmass=True)
    got = tot[idx]
    assert_bwd_close({"alpha": got[:, 0], "mu": got[:, 1:3], "sigma": got[:, 3:5],
                      "rho": got[:, 5], "color": got[:, 6:9]}, want, want["absmass"])
