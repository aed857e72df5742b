"""Per-rank cost of the row-band shard at G = 2, 4, 8, measured on ONE B200.

This run has one GPU, so the G-rank step is projected from measured parts: for every rank r of
G, the rank's whole per-step compute on the C5 batch (64 x 2040x1360, x8) is timed with CUDA
events exactly as bench.py's banded step runs it -- halo plan (K7 span pass over all N +
compaction), subset forward, subset backward moments, subset finalize, and the packing of the
seam buffers -- and the collective volumes are counted: the output all-gather (received bytes
per rank) and the neighbour seam exchange (sent bytes per rank). Projection (stated as such, not
a measurement): T_G = max_r compute_r + exchange_bytes / 770 GB/s (measured B200 peer copy,
B200_PROFILING.md) + 30 us per P2P pair + the part of the all-gather (770 GB/s) not hidden under
the rank's backward. The phase times per rank, the non-scaling part (halo plan + the O(N)
pieces) and the projected speedup over G = 1 are written as JSON.

usage: python tools/rank_projection.py [--images 64] [--iters 3] [--out profiles/r02_rank_projection.json]"""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import gsr_synth as S
import paper_2501_06838_b200 as gsr
from paper_2501_06838_b200 import dist as gd

KEYS = ("alpha", "mu", "sigma", "rho", "color")
PEER_GBS = 770.0
P2P_LAT_S = 30e-6


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=64)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--groups", default="1,2,4,8")
    ap.add_argument("--out", default="gpurun_out/r02_rank_projection.json")
    a = ap.parse_args()
    imgs = S.CONFIGS["C5"]["images"][:a.images]
    clouds = [S.gaussians(H, W, seed=1000 + k) for k, (H, W, s) in enumerate(imgs)]
    counts = [c["alpha"].shape[0] for c in clouds]
    offs = np.concatenate([[0], np.cumsum(counts)])
    dev = [torch.from_numpy(np.concatenate([c[k] for c in clouds])).cuda() for k in KEYS]
    n = int(offs[-1])
    whole = [(H, W, s, int(offs[k]), counts[k]) for k, (H, W, s) in enumerate(imgs)]
    dims = [gsr.out_dims(H, W, s) for H, W, s in imgs]
    widths3 = [w * 3 for _, w in dims]
    full_pix = sum(h * w for h, w in dims)
    res = {"workload": f"C5 first {len(imgs)} images", "n": n, "groups": {}}
    for G in [int(g) for g in a.groups.split(",")]:
        bounds = [gd.plan_bands(rc, G) for rc in gd.row_pair_counts(dev, whole, 0.1)]
        ranks = []
        for r in range(G):
            plan = gd.RankPlan(dev, whole, G, r, 0.1, bounds=bounds)
            lay = gsr.layout([gsr.Image(H, W, s, go, gc, rb, re)
                              for (H, W, s, go, gc, rb, re, sy) in plan.band_images()])
            g = torch.empty(lay.out_numel, device="cuda").uniform_(
                -1, 1, generator=torch.Generator(device="cuda").manual_seed(2000 + r))
            ws = gsr.subset_workspace_for(dev[0], lay, plan.m, 0.1)
            P_eval = gsr.pair_count(*dev, lay, 0.1, support=True)
            t = {k: [] for k in ("plan", "fwd", "bwd", "finalize", "pack", "total")}
            for it in range(a.iters + 1):
                e = [ev() for _ in range(6)]
                e[0].record()
                plan.refresh(dev)
                e[1].record()
                gsr.render_fwd_subset(*dev, plan.idx, lay, 0.1, workspace=ws)
                e[2].record()
                mom = torch.zeros((plan.m, 8), dtype=torch.float64, device="cuda")
                gsr.render_bwd_moments_subset(*dev, plan.idx, lay, g, mom, 0.1, workspace=ws,
                                              reuse_binning=True)
                e[3].record()
                comp = gsr.finalize_grads_subset(*dev, plan.idx, mom)
                e[4].record()
                cols = [c.view(plan.m, -1) for c in comp]
                for sel in (plan.up, plan.down):
                    if sel.numel():
                        torch.cat([c.index_select(0, sel) for c in cols], 1)
                e[5].record()
                torch.cuda.synchronize()
                if it == 0:
                    continue                         # warm-up
                for k, (i, j) in zip(("plan", "fwd", "bwd", "finalize", "pack", "total"),
                                     ((0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (0, 5))):
                    t[k].append(e[i].elapsed_time(e[j]))
            med = {k: statistics.median(v) for k, v in t.items()}
            xb = plan.exchange_bytes()
            numels = gd.rank_numels(bounds, widths3, G)
            gather_recv = 4 * max(numels) * (G - 1)
            ranks.append({"rank": r, "halo": plan.m, "halo_frac": plan.m / n,
                          "pairs_evaluated": P_eval, "ms": med, "exchange_bytes": xb,
                          "allgather_recv_bytes": gather_recv,
                          "band_rows_img0": [bounds[0][r], bounds[0][r + 1]]})
            del ws, mom, comp
        comp_max = max(x["ms"]["total"] for x in ranks)
        xmax = max(x["exchange_bytes"]["p2p_up"] + x["exchange_bytes"]["p2p_down"] +
                   x["exchange_bytes"]["multi_allreduce"] * 2 for x in ranks)
        t_x = xmax / (PEER_GBS * 1e9) * 1e3 + (2 * P2P_LAT_S * 1e3 if G > 1 else 0.0)
        ag = max(x["allgather_recv_bytes"] for x in ranks) / (PEER_GBS * 1e9) * 1e3
        hidden = min(x["ms"]["bwd"] for x in ranks)
        t_g = comp_max + t_x + max(0.0, ag - hidden)
        res["groups"][G] = {"ranks": ranks, "compute_max_ms": comp_max,
                            "exchange_ms_est": t_x, "allgather_ms_est": ag,
                            "allgather_exposed_ms_est": max(0.0, ag - hidden),
                            "non_scaling_ms_max": max(x["ms"]["plan"] + x["ms"]["pack"]
                                                      for x in ranks),
                            "projected_step_ms": t_g,
                            "projected_hr_mpix_per_s": full_pix / (t_g * 1e-3) / 1e6}
        print(f"G={G}: compute max {comp_max:.2f} ms (plan {max(x['ms']['plan'] for x in ranks):.2f}),"
              f" exchange {t_x:.2f} ms, all-gather {ag:.2f} ms (exposed "
              f"{max(0.0, ag - hidden):.2f}) -> projected {t_g:.2f} ms/step", flush=True)
    # baseline: the plain 1-GPU step of bench.py (no halo plan, all Gaussians binned)
    lay1 = gsr.layout([gsr.Image(H, W, s, go, gc) for (H, W, s, go, gc) in whole])
    g1 = torch.empty(lay1.out_numel, device="cuda").uniform_(-1, 1)
    from paper_2501_06838_b200 import ops
    ws1 = ops.workspace_for(dev[0], lay1, 0.1)
    ts = []
    for it in range(a.iters + 1):
        e0, e1 = ev(), ev()
        e0.record()
        gsr.render_fwd_batched(*dev, lay1, 0.1, workspace=ws1)
        mom = torch.zeros((n, 8), dtype=torch.float64, device="cuda")
        gsr.render_bwd_moments_batched(*dev, lay1, g1, mom, 0.1, workspace=ws1, reuse_binning=True)
        gsr.finalize_grads(*dev, mom)
        e1.record()
        torch.cuda.synchronize()
        if it:
            ts.append(e0.elapsed_time(e1))
    res["plain_1gpu_step_ms"] = statistics.median(ts)
    print(f"plain 1-GPU step {res['plain_1gpu_step_ms']:.2f} ms", flush=True)
    if res["groups"]:
        t1 = res["plain_1gpu_step_ms"]
        for G, v in res["groups"].items():
            v["projected_speedup_vs_plain_1gpu"] = t1 / v["projected_step_ms"]
    Path(a.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
