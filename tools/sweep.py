"""NEXT-3: the paper's rasterization-ratio and density sweeps as performance
workloads. 720x720 GT crops at x4 (LR 180x180) and x8 (LR 90x90), synthetic image-like
Gaussians (no weights needed), r in {0.01, 0.1, 0.4, 0.8, 1} at m = 16 (supp. Table)
and m in {1, 4, 9, 16} at r = 0.1. Reports forward (rendering-only, the quantity of
the paper's rendering-cost table) and forward+backward times with CUDA events, next to
the paper's A100 numbers where it has them.

usage: python tools/sweep.py [--out profiles/r01_sweep.json]"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import gsr_synth as S
import paper_2501_06838_b200 as gsr

# Paper numbers (single A100 per the cost protocol P:1725): rendering-only GSASR at
# r = 0.1, m = 16; whole-pipeline times of the r-ablation for the trend.
PAPER_RENDER_MS = {4: 168.0, 8: 71.0}
PAPER_PIPELINE_R_MS = {4: {0.01: 383, 0.1: 543, 0.4: 2490, 0.8: 6986, 1.0: 9419},
                       8: {0.01: 134, 0.1: 195, 0.4: 888, 0.8: 2451, 1.0: 3285}}


def time_case(H, W, s, m, r, reps=5):
    c = S.gaussians(H, W, m=m, seed=7)
    dev = [torch.from_numpy(c[k]).cuda() for k in ("alpha", "mu", "sigma", "rho", "color")]
    lay = gsr.layout([gsr.Image(H, W, s, 0, c["alpha"].shape[0])])
    P = gsr.pair_count(*dev, lay, r)
    g = torch.rand(lay.out_numel, device="cuda") * 2 - 1
    out = gsr.render_fwd_batched(*dev, lay, r)
    gsr.render_bwd_batched(*dev, lay, g, r)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf, tb = [], []
    for _ in range(reps):
        e[0].record()
        gsr.render_fwd_batched(*dev, lay, r, out=out)
        e[1].record()
        gsr.render_bwd_batched(*dev, lay, g, r)
        e[2].record()
        torch.cuda.synchronize()
        tf.append(e[0].elapsed_time(e[1]))
        tb.append(e[1].elapsed_time(e[2]))
    return dict(H=H, W=W, s=s, m=m, r=r, pairs=P, fwd_ms=float(np.median(tf)),
                bwd_ms=float(np.median(tb)), fwd_gpairs_s=P / np.median(tf) / 1e6,
                bwd_gpairs_s=P / np.median(tb) / 1e6)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    for s in (4, 8):
        H = W = 720 // s
        for r in (0.01, 0.1, 0.4, 0.8, 1.0):
            d = time_case(H, W, float(s), 16, r, reps=3 if r >= 0.4 else 5)
            d["paper_a100_pipeline_ms"] = PAPER_PIPELINE_R_MS[s][r]
            if r == 0.1:
                d["paper_a100_render_ms"] = PAPER_RENDER_MS[s]
            rows.append(d)
            print(json.dumps(d), flush=True)
        for m in (1, 4, 9):
            d = time_case(H, W, float(s), m, 0.1)
            rows.append(d)
            print(json.dumps(d), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps({"device": torch.cuda.get_device_name(),
                                              "lib": gsr.version(), "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
