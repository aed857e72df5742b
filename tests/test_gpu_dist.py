"""Row-band sharding through the real CUDA path with 2 ranks: two processes share
cuda:0 (this run has one GPU) and exchange over gloo. Each rank plans its bands and halo with
libgsr's K7 planner on the device (dist.RankPlan), renders its bands from its halo only
(render_fwd_subset), all-gathers them (dist.gather_bands), accumulates its halo's compact
moments (render_bwd_moments_subset), finalizes them (finalize_grads_subset) and swaps the seam
Gaussians' partial gradients with its neighbour (dist.exchange_seams). Checks: the gathered image equals the
single-process render of the same band layout bit for bit and the oracle within the forward
gate; after the seam reduce every Gaussian of the rank's halo and of the seam set has the
single-process whole-image gradient (fp32 regrouping tolerance) and sampled Gaussians match the
oracle (gate of tests/_util)."""
import os
import socket
from pathlib import Path

import numpy as np
import pytest

import gsr_synth as S
import oracle as O
from _util import KEYS, assert_bwd_close, assert_fwd_close

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

IMGS = [(40, 60, 8.0), (34, 51, 6.5)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs():
    clouds = [S.gaussians(H, W, seed=500 + k) for k, (H, W, s) in enumerate(IMGS)]
    counts = [c["alpha"].shape[0] for c in clouds]
    offs = np.concatenate([[0], np.cumsum(counts)])
    allc = {k: np.concatenate([c[k] for c in clouds]) for k in KEYS}
    return clouds, counts, offs, allc


def _worker(rank, world, port, outdir):
    import datetime
    import traceback
    try:
        _worker_body(rank, world, port, outdir)
    except BaseException:
        with open(os.path.join(outdir, f"rank{rank}.err"), "w") as f:
            f.write(traceback.format_exc())
        raise


def _worker_body(rank, world, port, outdir):
    import datetime
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world,
                            timeout=datetime.timedelta(seconds=120))
    try:
        import paper_2501_06838_b200 as gsr
        from paper_2501_06838_b200 import dist as gd
        torch.cuda.set_device(0)
        clouds, counts, offs, allc = _inputs()
        n = int(offs[-1])
        dev = [torch.from_numpy(allc[k]).cuda() for k in KEYS]
        whole = [(H, W, s, int(offs[k]), counts[k]) for k, (H, W, s) in enumerate(IMGS)]
        dims = [gsr.out_dims(H, W, s) for H, W, s in IMGS]
        widths3 = [w * 3 for _, w in dims]
        plan = gd.RankPlan(dev, whole, world, rank, 0.1)      # K7 on the device
        bounds = plan.bounds
        lay = gsr.layout([gsr.Image(H, W, s, go, gc, rb, re)
                          for (H, W, s, go, gc, rb, re, sy) in plan.band_images()])
        gfull = [torch.from_numpy(S.grad_out((h, w, 3), seed=600 + k)).cuda()
                 for k, (h, w) in enumerate(dims)]
        g_band = torch.cat([gfull[k][bounds[k][rank]:bounds[k][rank + 1]].reshape(-1)
                            for k in range(len(IMGS))])
        ws = gsr.subset_workspace_for(dev[0], lay, plan.m, 0.1)
        out = gsr.render_fwd_subset(*dev, plan.idx, lay, 0.1, workspace=ws)
        gathered, work = gd.gather_bands(out, gd.rank_numels(bounds, widths3, world),
                                         async_op=True)
        mom = torch.zeros((plan.m, 8), dtype=torch.float64, device="cuda")
        gsr.render_bwd_moments_subset(*dev, plan.idx, lay, g_band, mom, 0.1, workspace=ws,
                                      reuse_binning=True)
        comp = gsr.finalize_grads_subset(*dev, plan.idx, mom)
        gd.exchange_seams(comp, plan)
        work.wait()
        # scatter the compact gradients of the halo to global rows for the checks
        grads = [torch.zeros((n,) + tuple(t.shape[1:]), dtype=torch.float32, device="cuda")
                 for t in dev]
        for gg, cc in zip(grads, comp):
            gg.index_copy_(0, plan.idx.long(), cc)
        torch.cuda.synchronize()
        span = gd.band_spans(dev, whole, bounds, 0.1)
        halo = gd.halo_mask(span, rank)
        res = {"bounds": bounds, "seam": gd.seam_mask(span).cpu().numpy(),
               "halo": halo.cpu().numpy(),
               "grads": np.concatenate([t.view(n, -1).cpu().numpy() for t in grads], 1)}
        for k in range(len(IMGS)):
            res[f"img{k}"] = gd.assemble_image(gathered, bounds, widths3, k).cpu().numpy()
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), **{k: np.asarray(v) for k, v in
                                                               res.items() if k != "bounds"},
                 bounds=np.asarray(bounds))
    finally:
        dist.destroy_process_group()


def test_two_ranks_band_exchange_cuda(tmp_path):
    import torch
    import torch.multiprocessing as mp
    import paper_2501_06838_b200 as gsr
    ctx = mp.get_context("spawn")
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, str(tmp_path)), daemon=True)
          for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=300)
    for p in ps:
        if p.is_alive():
            p.kill()
    errs = [(tmp_path / f"rank{r}.err") for r in range(2)]
    msg = "\n".join(e.read_text() for e in errs if e.exists())
    assert all(p.exitcode == 0 for p in ps), f"{[p.exitcode for p in ps]}\n{msg}"
    R = [np.load(tmp_path / f"rank{r}.npz") for r in range(2)]

    clouds, counts, offs, allc = _inputs()
    n = int(offs[-1])
    dev = [torch.from_numpy(allc[k]).cuda() for k in KEYS]
    bounds = R[0]["bounds"].tolist()
    assert np.array_equal(R[1]["bounds"], R[0]["bounds"])
    dims = [gsr.out_dims(H, W, s) for H, W, s in IMGS]
    # single-process render of each rank's band layout (same images, tiles and split factor;
    # all Gaussians binned -- the halo subset visits the same Gaussians in the same order)
    # -> bit-exact
    widths3 = [w * 3 for _, w in dims]
    for r in range(2):
        lay = gsr.layout([gsr.Image(H, W, s, int(offs[k]), counts[k], bounds[k][r],
                                    bounds[k][r + 1]) for k, (H, W, s) in enumerate(IMGS)])
        ref = gsr.render_fwd_batched(*dev, lay, 0.1)
        for k in range(len(IMGS)):
            got = R[0][f"img{k}"][bounds[k][r]:bounds[k][r + 1]]
            assert np.array_equal(got, lay.view(ref, k).cpu().numpy().reshape(got.shape))
            assert np.array_equal(R[1][f"img{k}"], R[0][f"img{k}"])
    for k, (H, W, s) in enumerate(IMGS):
        want = O.render_fwd(clouds[k], H, W, s, 0.1)
        assert_fwd_close(R[0][f"img{k}"].reshape(want.shape), want)
    # gradients: halo and seam Gaussians carry the whole-image gradient after the seam reduce
    whole = gsr.layout([gsr.Image(H, W, s, int(offs[k]), counts[k])
                        for k, (H, W, s) in enumerate(IMGS)])
    gflat = torch.cat([torch.from_numpy(S.grad_out((h, w, 3), seed=600 + k)).reshape(-1)
                       for k, (h, w) in enumerate(dims)]).cuda()
    full = np.concatenate([t.view(n, -1).cpu().numpy() for t in
                           gsr.render_bwd_batched(*dev, whole, gflat, 0.1)], 1)
    scale = np.abs(full).max(0, keepdims=True)
    seam = R[0]["seam"]
    assert 0 < seam.sum() < n
    for r in range(2):
        sel = R[r]["halo"] | seam
        assert sel.sum() > 0
        assert (np.abs(R[r]["grads"][sel] - full[sel]) <= 1e-5 * scale).all()
        assert not R[r]["grads"][~sel].any()
    rng = np.random.default_rng(7)
    for k, (H, W, s) in enumerate(IMGS):
        loc = np.arange(counts[k])
        sk = seam[offs[k]:offs[k + 1]]
        idx = np.sort(np.concatenate([rng.choice(loc[sk], 10, replace=False),
                                      rng.choice(loc[~sk], 10, replace=False)]))
        g = S.grad_out((dims[k][0], dims[k][1], 3), seed=600 + k)
        want = O.render_bwd(clouds[k], H, W, s, 0.1, g, idx=idx, want_absmass=True)
        r = 0
        got = R[r]["grads"][offs[k] + idx]
        h = R[r]["halo"][offs[k] + idx] | sk[idx]
        got = np.where(h[:, None], got, R[1]["grads"][offs[k] + idx])
        assert_bwd_close({"alpha": got[:, 0], "mu": got[:, 1:3], "sigma": got[:, 3:5],
                          "rho": got[:, 5], "color": got[:, 6:9]}, want, want["absmass"])


@pytest.mark.parametrize("support", [False, True])
def test_k7_planner_device_equals_host_and_oracle(support):
    """gsr_row_pair_counts_batched / gsr_band_span_batched (device) == their _host variants ==
    the oracle, on a ragged batch with adversarial Gaussians (tile and window edges, outside,
    huge, invalid) and a scale vector."""
    import torch
    from paper_2501_06838_b200 import dist as gd
    from test_gpu_parity import adversarial_cloud
    spec = [(20, 33, 2.7, None), (9, 13, 30.0, None), (12, 10, 4.0, 2.5)]
    clouds = [adversarial_cloud(H, W, s, seed=k) for k, (H, W, s, sy) in enumerate(spec)]
    counts = [c["alpha"].shape[0] for c in clouds]
    offs = np.concatenate([[0], np.cumsum(counts)])
    allc = {k: np.concatenate([c[k] for c in clouds]) for k in KEYS}
    host = [allc[k] for k in KEYS]
    dev = [torch.from_numpy(a).cuda() for a in host]
    ims = [(H, W, s, int(offs[k]), counts[k], sy) for k, (H, W, s, sy) in enumerate(spec)]
    rd = gd.row_pair_counts(dev, ims, 0.1, support=support)
    rh = gd.row_pair_counts(host, ims, 0.1, support=support)
    for k, (H, W, s, sy) in enumerate(spec):
        assert np.array_equal(rd[k], rh[k])
        assert rd[k].sum() == O.pair_count(clouds[k], H, W, (s, sy) if sy else s, 0.1,
                                           support=support)
    bounds = [gd.plan_bands(r, 3) for r in rh]
    sd = gd.band_spans(dev, ims, bounds, 0.1, margin=1).cpu().numpy()
    sh = gd.band_spans(host, ims, bounds, 0.1, margin=1)
    assert np.array_equal(sd, sh)
    # bfloat16 parameters: the widened values give the float32 results
    rb = gd.row_pair_counts([t.bfloat16() for t in dev], ims, 0.1, support=support)
    rf = gd.row_pair_counts([t.bfloat16().float() for t in dev], ims, 0.1, support=support)
    assert all(np.array_equal(a, b) for a, b in zip(rb, rf))


def test_rank_halo_fused_equals_span_path():
    """gsr_rank_halo (the fused per-rank plan) == the plan built from gsr_band_span_batched with
    torch set operations, for every rank of G = 3 and 5 on a ragged batch incl. adversarial
    Gaussians (the multi-band path is exercised at r = 0.5)."""
    import torch
    from paper_2501_06838_b200 import dist as gd
    from test_gpu_parity import adversarial_cloud
    spec = [(20, 33, 2.7), (12, 18, 6.0), (16, 16, 4.0)]
    clouds = [adversarial_cloud(H, W, s, seed=k) for k, (H, W, s) in enumerate(spec)]
    counts = [c["alpha"].shape[0] for c in clouds]
    offs = np.concatenate([[0], np.cumsum(counts)])
    dev = [torch.from_numpy(np.concatenate([c[k] for c in clouds])).cuda() for k in KEYS]
    ims = [(H, W, s, int(offs[k]), counts[k]) for k, (H, W, s) in enumerate(spec)]
    for ratio in (0.1, 0.5):
        for G in (3, 5):
            for r in range(G):
                a = gd.RankPlan(dev, ims, G, r, ratio)                 # fused device path
                bnd = a.bounds
                b = gd.RankPlan.__new__(gd.RankPlan)
                b.world, b.rank, b.ratio, b.images, b.bounds = G, r, ratio, a.images, bnd
                gd.RankPlan.refresh(b, [t.cpu().numpy() for t in dev])   # span + torch path
                assert torch.equal(a.idx.cpu(), b.idx.to(torch.int32))
                for f in ("up", "down", "multi_pos", "multi_slot"):
                    assert torch.equal(getattr(a, f).cpu(), getattr(b, f).cpu()), f
                assert a.n_multi == b.n_multi
                if ratio == 0.5 and G == 5:
                    assert a.n_multi > 0


def _json_line(out: str) -> dict:
    import json
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_bench_self_launch_two_ranks():
    """`bench.py --gpus 2` with no launcher re-executes itself under torch.distributed.run (two
    ranks sharing cuda:0 over gloo here: GSR_BENCH_SHARE_GPU=1, a functional check of the
    sharded band path, never a performance number) and rank 0 prints one JSON line."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, GSR_BENCH_SHARE_GPU="1")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--images", "2",
                        "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--no-configs",
                        "--no-e2e"], capture_output=True, text=True, env=env, timeout=600,
                       cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    d = _json_line(r.stdout)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["halo_gaussians_rank0"] > 0


def test_train_dp_launcher_two_ranks():
    """NEXT-2's data-parallel launcher (tools/train_dp.py): two ranks, each its own 16 patches,
    the global-mean loss all-reduced (gloo on the shared GPU)."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, GSR_BENCH_SHARE_GPU="1")
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "train_dp.py"), "--gpus", "2",
                        "--steps", "3"], capture_output=True, text=True, env=env, timeout=600,
                       cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    d = _json_line(r.stdout)
    assert d["ranks"] == 2 and d["global_batch"] == 32 and d["global_mean_loss"] > 0
