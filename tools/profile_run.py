"""Runs one batched forward + backward of a config (for ncu captures).
usage: python tools/profile_run.py C5 [n_images]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import gsr_synth as S
import paper_2501_06838_b200 as gsr

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
nimg = int(sys.argv[2]) if len(sys.argv) > 2 else None
imgs = S.CONFIGS[name]["images"][:nimg] if nimg else S.CONFIGS[name]["images"]
clouds = [S.gaussians(H, W, seed=1000 + k) for k, (H, W, s) in enumerate(imgs)]
dev = [torch.from_numpy(np.concatenate([c[k] for c in clouds])).cuda()
       for k in ("alpha", "mu", "sigma", "rho", "color")]
ims, off = [], 0
for (H, W, s), c in zip(imgs, clouds):
    ims.append(gsr.Image(H, W, s, off, c["alpha"].shape[0]))
    off += c["alpha"].shape[0]
lay = gsr.layout(ims)
g = torch.rand(lay.out_numel, device="cuda") * 2 - 1
out = gsr.render_fwd_batched(*dev, lay)
grads = gsr.render_bwd_batched(*dev, lay, g)
torch.cuda.synchronize()
print("done", name, len(imgs), "P =", gsr.pair_count(*dev, lay))
