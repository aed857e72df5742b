"""Quick per-config timing of fwd / bwd (CUDA events), for development."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import gsr_synth as S
import paper_2501_06838_b200 as gsr

KEYS = ("alpha", "mu", "sigma", "rho", "color")


def run(name, nimg_override=None, iters=3):
    cfg = S.CONFIGS[name]
    imgs = cfg["images"] if nimg_override is None else cfg["images"][:nimg_override]
    clouds = [S.gaussians(H, W, seed=1000 + k) for k, (H, W, s) in enumerate(imgs)]
    dev = [torch.from_numpy(np.concatenate([c[k] for c in clouds])).cuda() for k in KEYS]
    ims, off = [], 0
    for (H, W, s), c in zip(imgs, clouds):
        ims.append(gsr.Image(H, W, s, off, c["alpha"].shape[0])); off += c["alpha"].shape[0]
    lay = gsr.layout(ims)
    Pw = gsr.pair_count(*dev, lay)
    try:
        P = gsr.pair_count(*dev, lay, support=True)     # evaluated pairs (reading R21)
    except Exception:                                   # an older library (A/B runs)
        P = Pw
    g = torch.rand(lay.out_numel, device="cuda") * 2 - 1
    out = gsr.render_fwd_batched(*dev, lay)
    gr = gsr.render_bwd_batched(*dev, lay, g)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf, tb = [], []
    for _ in range(iters):
        e[0].record(); gsr.render_fwd_batched(*dev, lay, out=out); e[1].record()
        gsr.render_bwd_batched(*dev, lay, g); e[2].record(); torch.cuda.synchronize()
        tf.append(e[0].elapsed_time(e[1])); tb.append(e[1].elapsed_time(e[2]))
    tf, tb = min(tf), min(tb)
    peak = 128 / 5.25 * 148 * 1.965e9      # forward, recurrence path (FP32 pipe)
    print(f"{name} imgs={len(imgs)} Pwin={Pw:.3e} Peval={P:.3e} fwd {tf:.3f} ms ({P/tf/1e9:.3f} Tpair/s, {P/tf*1e3/peak:.1%} of FP32) "
          f"bwd {tb:.3f} ms ({P/tb/1e9:.3f} Tpair/s, {P/tb*1e3/(128/12.5*148*1.965e9):.1%} of FP32)", flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:] or ["C1", "C2", "C4", "C3"]:
        if n == "C5s":
            run("C5", nimg_override=4, iters=2)
        else:
            run(n)
