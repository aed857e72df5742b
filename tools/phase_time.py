"""Per-phase timing of one step (binning, render_fwd, render_bwd, finalize) for development A/B:
CUDA-event phase times from libgsr's profiler (gsr_profile_enable/collect), median over iters.
The step is the bench's: forward (binning + K4), backward moments on the forward's binning (K5),
finalize (K6).  usage: python tools/phase_time.py C2 C5s ...   (GSR_LIB_PATH=... for A/B builds)"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import gsr_synth as S
import paper_2501_06838_b200 as gsr
from paper_2501_06838_b200 import ops
from paper_2501_06838_b200 import _lib

KEYS = ("alpha", "mu", "sigma", "rho", "color")


def run(name, nimg=None, iters=7):
    imgs = S.CONFIGS[name]["images"][:nimg] if nimg else S.CONFIGS[name]["images"]
    clouds = [S.gaussians(H, W, seed=1000 + k) for k, (H, W, s) in enumerate(imgs)]
    dev = [torch.from_numpy(np.concatenate([c[k] for c in clouds])).cuda() for k in KEYS]
    ims, off = [], 0
    for (H, W, s), c in zip(imgs, clouds):
        ims.append(gsr.Image(H, W, s, off, c["alpha"].shape[0])); off += c["alpha"].shape[0]
    lay = gsr.layout(ims)
    g = torch.rand(lay.out_numel, device="cuda") * 2 - 1
    ws = ops.workspace_for(dev[0], lay)
    out = torch.empty(lay.out_numel, device="cuda")
    mom = torch.zeros((off, 8), dtype=torch.float64, device="cuda")

    def step():
        ops.render_fwd_batched(*dev, lay, out=out, workspace=ws)
        mom.zero_()
        ops.render_bwd_moments_batched(*dev, lay, g, mom, workspace=ws, reuse_binning=True)
        return ops.finalize_grads(*dev, mom)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    res = {}
    for _ in range(iters):
        _lib.profile_collect(reset=True)
        _lib.profile_enable(True)
        step()
        torch.cuda.synchronize()
        _lib.profile_enable(False)
        ms, calls, _ = _lib.profile_collect(reset=True)
        for k, v in ms.items():
            res.setdefault(k, []).append(v)
    med = {k: float(np.median(v)) for k, v in res.items()}
    print(name, " ".join(f"{k} {v:.4f}" for k, v in med.items()), "sum %.4f ms" % sum(med.values()),
          flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:] or ["C1", "C2", "C4"]:
        if n == "C5s":
            run("C5", nimg=4, iters=3)
        else:
            run(n)
