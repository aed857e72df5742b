"""Forward error vs the oracle for the recurrence-regime cases (development diagnostic)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import gsr_synth as S
import oracle as O
import paper_2501_06838_b200 as gsr

KEYS = ("alpha", "mu", "sigma", "rho", "color")
for s, r, sig, dist in [(2.0, 0.6, 1.0, "image"), (3.0, 0.4, 1.0, "image"), (4.0, 0.3, 1.0, "image"),
                        (8.0, 0.3, 1.0, "image"), (4.0, 0.3, 0.5, "image"), (4.0, 0.3, 2.0, "image"),
                        (3.0, 0.4, 1.0, "stress"), (2.5, 0.5, 0.7, "stress")]:
    H = W = 24
    c = S.gaussians(H, W, m=4, seed=int(10 * s) + int(10 * sig), dist=dist)
    c["sigma"] = (c["sigma"] * np.float32(sig)).astype(np.float32)
    got = gsr.render_fwd(*[torch.from_numpy(c[k]).cuda() for k in KEYS], H, W, s, ratio=r).cpu().numpy()
    want = O.render_fwd(c, H, W, s, r, mode="rect")
    err = np.abs(got - want)
    rel = err / np.maximum(1.0, np.abs(want))
    print(f"s={s} r={r} sig={sig} {dist}: max abs {err.max():.2e} max rel {rel.max():.2e} "
          f"max|I| {np.abs(want).max():.2f}")
