"""Debug: K7 device planner on one process (no collectives)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import gsr_synth as S
import paper_2501_06838_b200 as gsr
from paper_2501_06838_b200 import dist as gd
KEYS = ("alpha", "mu", "sigma", "rho", "color")
c = S.gaussians(40, 60, seed=1)
host = [c[k] for k in KEYS]
dev = [torch.from_numpy(a).cuda() for a in host]
ims = [(40, 60, 8.0, 0, c["alpha"].shape[0])]
t = time.time()
rd = gd.row_pair_counts(dev, ims, 0.1); torch.cuda.synchronize()
print("row counts dev ok", time.time() - t, rd[0].sum(), flush=True)
rh = gd.row_pair_counts(host, ims, 0.1)
print("host == dev", np.array_equal(rd[0], rh[0]), flush=True)
b = [gd.plan_bands(rd[0], 2)]
sp = gd.band_spans(dev, ims, b, 0.1); torch.cuda.synchronize()
print("span dev ok", sp.shape, flush=True)
sh = gd.band_spans(host, ims, b, 0.1)
print("span host == dev", np.array_equal(sp.cpu().numpy(), sh), flush=True)
