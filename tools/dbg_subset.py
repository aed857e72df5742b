"""Debug: subset-mode forward vs plain forward (bit-exactness, timing)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import gsr_synth as S
import paper_2501_06838_b200 as gsr
from paper_2501_06838_b200 import dist as gd, ops
KEYS = ("alpha", "mu", "sigma", "rho", "color")
imgs = S.CONFIGS["C5"]["images"][:4]
clouds = [S.gaussians(H, W, seed=1000 + k) for k, (H, W, s) in enumerate(imgs)]
counts = [c["alpha"].shape[0] for c in clouds]
offs = np.concatenate([[0], np.cumsum(counts)])
dev = [torch.from_numpy(np.concatenate([c[k] for c in clouds])).cuda() for k in KEYS]
n = int(offs[-1])
whole = [(H, W, s, int(offs[k]), counts[k]) for k, (H, W, s) in enumerate(imgs)]
lay = gsr.layout([gsr.Image(H, W, s, go, gc) for (H, W, s, go, gc) in whole])
def timeit(fn, it=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): r = fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it, r
ws = ops.workspace_for(dev[0], lay, 0.1)
t0, a = timeit(lambda: gsr.render_fwd_batched(*dev, lay, 0.1, workspace=ws).clone())
print("plain", t0)
for name, idx in [("arange", torch.arange(n, dtype=torch.int32, device="cuda")),
                  ("plan", gd.RankPlan(dev, whole, 1, 0, 0.1).idx)]:
    wss = gsr.subset_workspace_for(dev[0], lay, idx.numel(), 0.1)
    t1, b = timeit(lambda: gsr.render_fwd_subset(*dev, idx, lay, 0.1, workspace=wss).clone())
    d = (a - b).abs()
    print(name, "m", idx.numel(), "ms", t1, "bitexact", bool(torch.equal(a, b)), "maxdiff", float(d.max()),
          "ndiff", int((d > 0).sum()), "sorted", bool((idx[1:] > idx[:-1]).all()))
