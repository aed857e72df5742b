"""One forward + backward of a small workload through the C-ABI, for compute-sanitizer runs
(racecheck / synccheck / memcheck) of libgsr's kernels: C1 (cluster split-K forward + DSMEM
reduce, split backward), C2 (ragged 16-patch batch, small-tile forward), a C5 band (the large
configuration, recurrence path, 64-row band of one image), a subset (halo) call, and chunks (a
dense image with very wide supports, r = 1: the forward's candidate stream over > 32 cell rows,
rebuilt under CTA barriers, trimmed by the cell reach).
usage: python tools/sanitize_run.py C1|C2|C5band|subset|chunks"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import gsr_synth as S
import paper_2501_06838_b200 as gsr
from paper_2501_06838_b200 import dist as gd

KEYS = ("alpha", "mu", "sigma", "rho", "color")
name = sys.argv[1]
if name == "C1":
    imgs, rows = [(48, 48, 4.0)], None
elif name == "C2":
    imgs, rows = [(48, 48, float(s)) for s in S.c2_scales()], None
elif name == "chunks":
    imgs, rows = [(40, 60, 8.0)], None
else:
    imgs, rows = [(170, 255, 8.0)], (600, 664)
ratio = 1.0 if name == "chunks" else 0.1
clouds = [S.gaussians(H, W, seed=1000 + k) for k, (H, W, s) in enumerate(imgs)]
if name == "chunks":
    clouds[0]["sigma"][::50] = 3.0
counts = [c["alpha"].shape[0] for c in clouds]
offs = np.concatenate([[0], np.cumsum(counts)])
dev = [torch.from_numpy(np.concatenate([c[k] for c in clouds])).cuda() for k in KEYS]
if rows:
    lay = gsr.layout([gsr.Image(H, W, s, int(offs[k]), counts[k], rows[0], rows[1])
                      for k, (H, W, s) in enumerate(imgs)])
else:
    lay = gsr.layout([gsr.Image(H, W, s, int(offs[k]), counts[k])
                      for k, (H, W, s) in enumerate(imgs)])
g = torch.empty(lay.out_numel, device="cuda").uniform_(-1, 1)
if name == "subset":
    whole = [(H, W, s, int(offs[k]), counts[k]) for k, (H, W, s) in enumerate(imgs)]
    plan = gd.RankPlan(dev, whole, 4, 1, 0.1)
    lay = gsr.layout([gsr.Image(H, W, s, go, gc, rb, re)
                      for (H, W, s, go, gc, rb, re, sy) in plan.band_images()])
    g = torch.empty(lay.out_numel, device="cuda").uniform_(-1, 1)
    ws = gsr.subset_workspace_for(dev[0], lay, plan.m, 0.1)
    out = gsr.render_fwd_subset(*dev, plan.idx, lay, 0.1, workspace=ws)
    mom = torch.zeros((plan.m, 8), dtype=torch.float64, device="cuda")
    gsr.render_bwd_moments_subset(*dev, plan.idx, lay, g, mom, 0.1, workspace=ws,
                                  reuse_binning=True)
    grads = gsr.finalize_grads_subset(*dev, plan.idx, mom)
else:
    out = gsr.render_fwd_batched(*dev, lay, ratio)
    grads = gsr.render_bwd_batched(*dev, lay, g, ratio)
torch.cuda.synchronize()
print(name, "ok", float(out.abs().sum()), float(grads[0].abs().sum()))
