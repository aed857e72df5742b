"""Host logic of the multi-GPU row-band path (paper_2501_06838_b200/dist.py) on CPU: band
planning against the oracle's pair counts, and the collective assembly with world_size 2 over
gloo, with the float64 oracle as the band renderer stand-in (the CUDA kernels need a GPU)."""
import os
import socket

import numpy as np
import pytest

import gsr_synth as S
import oracle as O
from paper_2501_06838_b200 import dist as gd


def test_row_pair_counts_match_oracle():
    for (H, W, s) in [(20, 25, 3.0), (9, 14, 8.0), (12, 12, 2.5)]:
        c = S.gaussians(H, W, seed=3, offset_range=1.5)
        rc = gd.row_pair_counts(c["mu"], np.ones(c["alpha"].shape[0], bool), H, W, s, 0.1)
        Hs, _ = O.out_dims(H, W, s)
        assert rc.shape == (Hs,)
        assert rc.sum() == O.pair_count(c, H, W, s, 0.1)
        for rb, re in [(0, 5), (7, 19), (Hs - 3, Hs)]:
            assert rc[rb:re].sum() == O.pair_count(c, H, W, s, 0.1, rows=(rb, re))
        # support rects (reading R21): the pairs the kernels evaluate
        rs = gd.row_pair_counts(c["mu"], np.ones(c["alpha"].shape[0], bool), H, W, s, 0.3,
                                sigma=c["sigma"])
        assert rs.sum() == O.pair_count(c, H, W, s, 0.3, support=True)
        assert rs[7:19].sum() == O.pair_count(c, H, W, s, 0.3, rows=(7, 19), support=True)


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_plan_bands_balanced(G):
    H, W, s = 34, 51, 8.0                        # C5 geometry scaled down 5x
    c = S.gaussians(H, W, seed=1)
    rc = gd.row_pair_counts(c["mu"], np.ones(c["alpha"].shape[0], bool), H, W, s, 0.1)
    b = gd.plan_bands(rc, G)
    assert b[0] == 0 and b[-1] == rc.shape[0] and len(b) == G + 1
    assert all(b[i] < b[i + 1] for i in range(G))
    # equal-row bands are ~5% imbalanced at G = 8; pair-balanced bands are
    # within one row's worth of work of perfect
    row_max = rc.max() / (rc.sum() / G)
    assert gd.band_imbalance(rc, b) <= 1.0 + row_max + 1e-9
    eq = [round(g * rc.shape[0] / G) for g in range(G + 1)]
    assert gd.band_imbalance(rc, b) <= gd.band_imbalance(rc, eq) + 1e-9


def test_plan_bands_degenerate():
    assert gd.plan_bands(np.zeros(5, np.int64), 4) == [0, 1, 2, 3, 5]
    b = gd.plan_bands(np.ones(3, np.int64), 8)           # more ranks than rows
    assert b[0] == 0 and b[-1] == 3 and all(b[i] <= b[i + 1] for i in range(8))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_support_rows_match_oracle_and_seams():
    """support_rows reproduces the oracle's support rects (R21) row for row; the seam set is
    exactly the Gaussians whose rows meet two bands (margin 0) and contains them (margin 1)."""
    for (H, W, s, sv) in [(20, 25, 3.0, None), (9, 14, 8.0, None), (12, 10, 4.0, 2.5)]:
        c = S.gaussians(H, W, seed=5, offset_range=1.5)
        n = c["alpha"].shape[0]
        valid = np.ones(n, bool)
        y0, y1, ok = gd.support_rows(c["mu"], c["sigma"], valid, H, W, s, 0.1, s_y=sv)
        R = O.rects(c, H, W, (s, sv) if sv else s, 0.1, support=True)
        nonempty = (R[:, 2] <= R[:, 3]) & (R[:, 4] <= R[:, 5])
        assert np.array_equal(ok, nonempty)
        assert np.array_equal(y0[ok], R[ok, 4]) and np.array_equal(y1[ok], R[ok, 5])
        Hs = O.out_dims(H, W, (s, sv) if sv else s)[0]
        b = [0, Hs // 3, (2 * Hs) // 3 + 1, Hs]
        exact = gd.seam_mask(c["mu"], c["sigma"], valid, H, W, s, 0.1, b, margin=0, s_y=sv)
        bands = [gd.halo_mask(c["mu"], c["sigma"], valid, H, W, s, 0.1, (b[g], b[g + 1]), s_y=sv)
                 for g in range(3)]
        assert np.array_equal(exact, np.sum(bands, 0) >= 2)
        wide = gd.seam_mask(c["mu"], c["sigma"], valid, H, W, s, 0.1, b, margin=1, s_y=sv)
        assert not (exact & ~wide).any() and 0 < exact.sum() < n


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        imgs = [(10, 12, 3.0), (8, 9, 2.5)]
        clouds = [S.gaussians(H, W, seed=40 + k) for k, (H, W, s) in enumerate(imgs)]
        counts = [c["alpha"].shape[0] for c in clouds]
        offs = np.concatenate([[0], np.cumsum(counts)])
        n = int(offs[-1])
        dims = [O.out_dims(H, W, s) for H, W, s in imgs]
        widths3 = [w * 3 for _, w in dims]
        bounds = []
        for (H, W, s), c in zip(imgs, clouds):
            rc = gd.row_pair_counts(c["mu"], np.ones(c["alpha"].shape[0], bool), H, W, s, 0.1)
            bounds.append(gd.plan_bands(rc, world))
        grads_full = [S.grad_out((h, w, 3), seed=7 + k) for k, (h, w) in enumerate(dims)]

        def render_band(rows):
            parts = [O.render_fwd(c, H, W, s, 0.1, rows=r).reshape(-1)
                     for (H, W, s), c, r in zip(imgs, clouds, rows)]
            return torch.from_numpy(np.concatenate(parts))

        def moments_band(rows, mom):
            for k, ((H, W, s), c, (rb, re)) in enumerate(zip(imgs, clouds, rows)):
                if re <= rb:
                    continue
                # support mode (R21): the pairs the kernels evaluate, so a Gaussian outside the
                # band's support halo has exactly zero moments there
                d = O.render_bwd(c, H, W, s, 0.1, grads_full[k][rb:re], rows=(rb, re),
                                 mode="support")
                blk = np.concatenate([d["alpha"][:, None], d["mu"], d["sigma"], d["rho"][:, None],
                                      d["color"]], 1)
                mom[offs[k]:offs[k + 1]] += torch.from_numpy(blk)

        seam = np.concatenate([gd.seam_mask(c["mu"], c["sigma"], np.ones(cn, bool), H, W, s,
                                            0.1, b)
                               for (H, W, s), c, cn, b in zip(imgs, clouds, counts, bounds)])
        halo = np.concatenate([gd.halo_mask(c["mu"], c["sigma"], np.ones(cn, bool), H, W, s, 0.1,
                                            (b[rank], b[rank + 1]))
                               for (H, W, s), c, cn, b in zip(imgs, clouds, counts, bounds)])
        ok = bool(0 < seam.sum() < n)
        for seam_idx in (torch.from_numpy(np.nonzero(seam)[0]), None):
            gathered, grads = gd.sharded_step(rank, world, bounds, widths3, render_band,
                                              moments_band, lambda m: m, n, "cpu", moment_cols=9,
                                              seam_idx=seam_idx)
            for k, ((H, W, s), c) in enumerate(zip(imgs, clouds)):
                full = gd.assemble_image(gathered, bounds, widths3, k).numpy()
                ref = O.render_fwd(c, H, W, s, 0.1).reshape(dims[k][0], -1)
                ok &= bool(np.array_equal(full, ref))
                d = O.render_bwd(c, H, W, s, 0.1, grads_full[k], mode="support")
                blk = np.concatenate([d["alpha"][:, None], d["mu"], d["sigma"],
                                      d["rho"][:, None], d["color"]], 1)
                got = grads[offs[k]:offs[k + 1]].numpy()
                # seam reduce: final gradients for the rank's halo (and every seam Gaussian),
                # 0 elsewhere; full: all
                sel = halo[offs[k]:offs[k + 1]] if seam_idx is not None else slice(None)
                ok &= bool(np.allclose(got[sel], blk[sel], rtol=1e-12, atol=1e-13))
                if seam_idx is not None:      # neither in the halo nor reduced: untouched zeros
                    rest = ~(halo | seam)[offs[k]:offs[k + 1]]
                    ok &= bool(rest.any() and not got[rest].any())
                    both = (halo | seam)[offs[k]:offs[k + 1]]
                    ok &= bool(np.allclose(got[both], blk[both], rtol=1e-12, atol=1e-13))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_sharded_step_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)]
