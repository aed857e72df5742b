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


def P(c):
    return [c[k] for k in ("alpha", "mu", "sigma", "rho", "color")]


def test_row_pair_counts_match_oracle():
    """K7 planner of libgsr (host variant, the kernels' rect code) vs the oracle's pair counts:
    window rects (Alg. 1) and support rects (R21), whole images and row ranges, a ragged
    batch of three images in one call, a scale vector, and invalid Gaussians (R20)."""
    imgs = [(20, 25, 3.0, None), (9, 14, 8.0, None), (12, 12, 2.5, None), (12, 10, 4.0, 2.5)]
    clouds = [S.gaussians(H, W, seed=3 + k, offset_range=1.5) for k, (H, W, s, sy) in
              enumerate(imgs)]
    clouds[1]["sigma"][3, 0] = 0.0                        # invalid (R20)
    clouds[2]["rho"][5] = np.float32(1.0)
    allc = {k: np.concatenate([c[k] for c in clouds]) for k in clouds[0]}
    offs = np.concatenate([[0], np.cumsum([c["alpha"].shape[0] for c in clouds])])
    ims = [(H, W, s, int(offs[k]), int(offs[k + 1] - offs[k]), sy)
           for k, (H, W, s, sy) in enumerate(imgs)]
    for r, support in [(0.1, False), (0.3, True), (0.1, True)]:
        rcs = gd.row_pair_counts(P(allc), ims, r, support=support)
        for (H, W, s, sy), c, rc in zip(imgs, clouds, rcs):
            sv = (s, sy) if sy else s
            Hs, _ = O.out_dims(H, W, sv)
            assert rc.shape == (Hs,)
            assert rc.sum() == O.pair_count(c, H, W, sv, r, support=support)
            for rb, re in [(0, 5), (7, 19), (Hs - 3, Hs)]:
                assert rc[rb:re].sum() == O.pair_count(c, H, W, sv, r, rows=(rb, re),
                                                       support=support)


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_plan_bands_balanced(G):
    H, W, s = 34, 51, 8.0                        # C5 geometry scaled down 5x
    c = S.gaussians(H, W, seed=1)
    rc = gd.row_pair_counts(P(c), [(H, W, s, 0, c["alpha"].shape[0])], 0.1)[0]
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


def test_band_spans_match_oracle_and_seams():
    """K7 band spans (host variant) vs the oracle's support rects (R21): first/last band met by
    every Gaussian's support rows; the seam set is exactly the Gaussians whose rows meet two
    bands, halos are the Gaussians meeting a band, and a margin only widens the seam set."""
    for (H, W, s, sv) in [(20, 25, 3.0, None), (9, 14, 8.0, None), (12, 10, 4.0, 2.5)]:
        c = S.gaussians(H, W, seed=5, offset_range=1.5)
        c["alpha"][0] = np.float32(np.nan)                 # invalid (R20): no span
        n = c["alpha"].shape[0]
        R = O.rects(c, H, W, (s, sv) if sv else s, 0.1, support=True)
        nonempty = (R[:, 2] <= R[:, 3]) & (R[:, 4] <= R[:, 5])
        Hs = O.out_dims(H, W, (s, sv) if sv else s)[0]
        b = [0, Hs // 3, (2 * Hs) // 3 + 1, Hs]
        ims = [(H, W, s, 0, n, sv)]
        span = gd.band_spans(P(c), ims, [b], 0.1, margin=0)
        assert np.array_equal(span[:, 0] >= 0, nonempty)
        band = lambda y: np.searchsorted(np.asarray(b), y, side="right") - 1
        assert np.array_equal(span[nonempty, 0], band(R[nonempty, 4]))
        assert np.array_equal(span[nonempty, 1], band(R[nonempty, 5]))
        exact = gd.seam_mask(span)
        halos = [gd.halo_mask(span, g) for g in range(3)]
        for g in range(3):
            meets = nonempty & (R[:, 5] >= b[g]) & (R[:, 4] < b[g + 1])
            assert np.array_equal(halos[g], meets)
        assert np.array_equal(exact, np.sum(halos, 0) >= 2)
        wide = gd.seam_mask(gd.band_spans(P(c), ims, [b], 0.1, margin=1))
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
        allc = {k: np.concatenate([c[k] for c in clouds]) for k in clouds[0]}
        ims = [(H, W, s, int(offs[k]), counts[k]) for k, (H, W, s) in enumerate(imgs)]
        bounds = [gd.plan_bands(rc, world) for rc in gd.row_pair_counts(P(allc), ims, 0.1)]
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

        span = gd.band_spans(P(allc), ims, bounds, 0.1)
        seam = gd.seam_mask(span)
        halo = gd.halo_mask(span, rank)
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


def _worker_subset(rank, world, port, q):
    """Subset mode + neighbour seam exchange (dist.RankPlan / exchange_seams) with the oracle as
    the band renderer: each rank computes the compact partial gradients of its halo over its
    own bands only; after the exchange every halo Gaussian has its whole-image gradient."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        imgs = [(12, 14, 3.0), (9, 11, 4.0)]          # small bands: some supports span 3 bands
        clouds = [S.gaussians(H, W, seed=70 + k) for k, (H, W, s) in enumerate(imgs)]
        counts = [c["alpha"].shape[0] for c in clouds]
        offs = np.concatenate([[0], np.cumsum(counts)])
        allc = {k: np.concatenate([c[k] for c in clouds]) for k in clouds[0]}
        ims = [(H, W, s, int(offs[k]), counts[k]) for k, (H, W, s) in enumerate(imgs)]
        r_ = 0.5 if world == 3 else 0.1       # r = 0.5: windows taller than a band
        plan = gd.RankPlan(P(allc), ims, world, rank, r_)
        idx = plan.idx.numpy().astype(np.int64)
        dims = [O.out_dims(H, W, s) for H, W, s in imgs]
        gfull = [S.grad_out((h, w, 3), seed=80 + k) for k, (h, w) in enumerate(dims)]
        part = np.zeros((idx.size, 9))
        full = np.zeros((idx.size, 9))
        for k, ((H, W, s), c) in enumerate(zip(imgs, clouds)):
            sel = (idx >= offs[k]) & (idx < offs[k + 1])
            loc = idx[sel] - offs[k]
            if loc.size == 0:
                continue
            rb, re = plan.bounds[k][rank], plan.bounds[k][rank + 1]
            d = O.render_bwd(c, H, W, s, r_, gfull[k][rb:re], rows=(rb, re), mode="support",
                             idx=loc)
            part[sel] = np.concatenate([d["alpha"][:, None], d["mu"], d["sigma"],
                                        d["rho"][:, None], d["color"]], 1)
            d = O.render_bwd(c, H, W, s, r_, gfull[k], mode="support", idx=loc)
            full[sel] = np.concatenate([d["alpha"][:, None], d["mu"], d["sigma"],
                                        d["rho"][:, None], d["color"]], 1)
        G = torch.from_numpy(part.copy())
        gd.exchange_seams(G, plan)
        ok = bool(np.allclose(G.numpy(), full, rtol=1e-12, atol=1e-14))
        ok &= (plan.up.numel() + plan.down.numel()) > 0
        ok &= world < 3 or plan.n_multi > 0          # 3 bands: the multi-band path is exercised
        q.put((rank, ok, plan.n_multi))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_subset_neighbour_exchange_gloo(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_subset, args=(r, world, port, q), daemon=True)
          for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
