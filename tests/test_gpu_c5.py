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


def test_c5_full_size_sampled():
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


def test_band_partials_and_seam_set():
    """The row-band exchange of dist.py on the CUDA path, emulated in one process (this run has
    one GPU): G = 4 pair-balanced bands of a C5-geometry image; each band's moments are
    finalized on their own (the finalize is linear in the moments); a Gaussian outside the seam
    set has a nonzero partial in at most one band, where it equals the oracle's gradient; the
    band partials summed over the seam set equal the whole-image gradients."""
    import torch
    import paper_2501_06838_b200 as gsr
    from paper_2501_06838_b200 import dist as gd
    H, W, s, G = 60, 90, 8.0, 4
    c = S.gaussians(H, W, seed=77)
    n = c["alpha"].shape[0]
    dev = [torch.from_numpy(c[k]).cuda() for k in KEYS]
    valid = np.ones(n, bool)
    rc = gd.row_pair_counts(c["mu"], valid, H, W, s, 0.1, sigma=c["sigma"])
    b = gd.plan_bands(rc, G)
    seam = gd.seam_mask(c["mu"], c["sigma"], valid, H, W, s, 0.1, b)
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
