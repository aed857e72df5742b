"""NEXT-2: the paper's real training batch shapes through the fused training step
(activations -> render -> L1 loss -> raw gradients, ops.train_step_l1), timed with CUDA events:

  * EDSR/RDN training slice: 16 LR patches of 48x48 per GPU, per-patch scale
    s ~ U[1, 4], m = 16 Gaussians per LR pixel;
  * HAT-L variant: 8 patches of 64x64 per GPU, s ~ U[1, 16].

For each: direct launches with a fixed scale draw, the same step replayed from a CUDA graph
(ops.TrainStepGraph), and direct launches with a new scale draw every step (the training loop's
real pattern: a new layout per step, so a graph would have to be re-captured). Synthetic raw
head outputs (gsr_synth's image-like recipe before activation) and a random ground truth.

usage: python tools/train_bench.py [--steps 30] [--out profiles/r01_train_bench.json]"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import gsr_synth as S
import paper_2501_06838_b200 as gsr
from paper_2501_06838_b200 import ops

M = 16
ORDER = ("raw_alpha", "offset", "ref", "raw_sigma", "raw_rho", "raw_color")


def batch(B, P, smax, seed):
    rng = np.random.default_rng(seed)
    scales = rng.uniform(1.0, smax, B)
    n1 = M * P * P
    n = B * n1
    ref = np.concatenate([S.reference_grid(P, P, M) for _ in range(B)]).astype(np.float32)
    raw = dict(raw_alpha=rng.normal(-3, 1, n), offset=rng.uniform(-0.5, 0.5, (n, 2)),
               raw_sigma=rng.normal(-0.5, 0.5, (n, 2)), raw_rho=rng.normal(0, 0.5, n),
               raw_color=rng.normal(0, 1, (n, 3)))
    dev = {k: torch.from_numpy(v.astype(np.float32)).cuda() for k, v in raw.items()}
    dev["ref"] = torch.from_numpy(ref).cuda()
    return dev, scales, n1


def layout_for(B, P, scales, n1):
    return gsr.layout([gsr.Image(P, P, float(s), k * n1, n1) for k, s in enumerate(scales)])


def timed(fn, steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def run(name, B, P, smax, steps):
    dev, scales, n1 = batch(B, P, smax, seed=7)
    lay = layout_for(B, P, scales, n1)
    gt = torch.rand(lay.out_numel, device="cuda")
    args = [dev[k] for k in ORDER]
    direct = timed(lambda: ops.train_step_l1(*args, lay, gt), steps)
    g = gsr.TrainStepGraph(lay, B * n1)
    graph = timed(lambda: g(*args, gt), steps)
    # correctness of the replay against the direct call
    out_d, loss_d, gr_d = ops.train_step_l1(*args, lay, gt)
    out_g, loss_g, gr_g = g(*args, gt)
    torch.cuda.synchronize()
    same = (torch.allclose(out_d, out_g, rtol=1e-6, atol=1e-7) and
            abs(loss_d.item() - loss_g.item()) <= 1e-9 * max(1.0, abs(loss_d.item())))
    rng = np.random.default_rng(11)
    gts = {}

    def varying():
        sc = rng.uniform(1.0, smax, B)
        ly = layout_for(B, P, sc, n1)
        if ly.out_numel not in gts:
            gts[ly.out_numel] = torch.rand(ly.out_numel, device="cuda")
        ops.train_step_l1(*args, ly, gts[ly.out_numel])
    vary = timed(varying, steps)
    hr_px = lay.out_numel / 3
    res = dict(workload=name, patches=B, lr=P, s_max=smax, gaussians=B * n1,
               hr_px_per_step=int(hr_px), direct_ms=direct, graph_ms=graph,
               varying_scales_ms=vary, graph_matches_direct=bool(same),
               patches_per_s_graph=B / (graph * 1e-3),
               hr_mpix_per_s_graph=hr_px / (graph * 1e-3) / 1e6)
    print(json.dumps(res), flush=True)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = [run("EDSR/RDN slice: 16 x 48x48, s~U[1,4]", 16, 48, 4.0, a.steps),
            run("HAT-L slice: 8 x 64x64, s~U[1,16]", 8, 64, 16.0, a.steps)]
    if a.out:
        Path(a.out).write_text(json.dumps({"device": torch.cuda.get_device_name(),
                                           "lib": gsr.version(), "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
