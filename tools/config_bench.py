"""Per-config timing of the hot path on every BASELINE.json configuration (SURVEY 8(d) timing
protocol): CUDA events, >= 5 warm-ups, median of 20 iterations; one step = forward (binning +
K4) + backward (K5 reusing the forward's binning + K6), device-resident inputs. C1/C2 (the small
training-size problems) are also captured once in a CUDA graph and replayed. Reports evaluated
pairs per second and the fraction of the FP32-pipe rooflines of DESIGN.md section 7.

usage: python tools/config_bench.py [--iters 20] [--out profiles/r01_configs.json]"""
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
from paper_2501_06838_b200 import ops

KEYS = ("alpha", "mu", "sigma", "rho", "color")
CLK, SMS = 1.965e9, 148
PEAK_FWD = 128 / 5.25 * SMS * CLK        # recurrence path, pairs/s
PEAK_BWD = 128 / 12.5 * SMS * CLK


def median_ms(fn, iters, warmup=5):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def run(name, iters, quiet=False):
    cfg = S.CONFIGS["C5" if name == "C5s" else name]
    imgs = cfg["images"][:4] if name == "C5s" else cfg["images"]     # C5s: a 4-image slice
    clouds = [S.gaussians(H, W, seed=1000 + k) for k, (H, W, s) in enumerate(imgs)]
    dev = [torch.from_numpy(np.concatenate([c[k] for c in clouds])).cuda() for k in KEYS]
    ims, off = [], 0
    for (H, W, s), c in zip(imgs, clouds):
        ims.append(gsr.Image(H, W, s, off, c["alpha"].shape[0]))
        off += c["alpha"].shape[0]
    lay = gsr.layout(ims)
    n = off
    P_win = gsr.pair_count(*dev, lay)
    P = gsr.pair_count(*dev, lay, support=True)
    ws = ops.workspace_for(dev[0], lay)
    out = torch.empty(lay.out_numel, device="cuda")
    g = torch.empty(lay.out_numel, device="cuda").uniform_(
        -1, 1, generator=torch.Generator(device="cuda").manual_seed(2000))
    mom = torch.zeros((n, 8), dtype=torch.float64, device="cuda")

    def fwd():
        gsr.render_fwd_batched(*dev, lay, out=out, workspace=ws)

    def bwd():
        mom.zero_()
        gsr.render_bwd_moments_batched(*dev, lay, g, mom, workspace=ws, reuse_binning=True)
        return gsr.finalize_grads(*dev, mom)

    def step():
        fwd()
        bwd()

    t_fwd = median_ms(fwd, iters)
    t_step = median_ms(step, iters)
    t_bwd = t_step - t_fwd
    row = dict(config=name, desc=cfg.get("desc", ""), images=len(imgs), gaussians=n,
               hr_px=lay.out_numel // 3, pairs_window=P_win, pairs_evaluated=P,
               fwd_ms=t_fwd, bwd_ms=t_bwd, step_ms=t_step,
               fwd_frac=P / (t_fwd * 1e-3) / PEAK_FWD, bwd_frac=P / (t_bwd * 1e-3) / PEAK_BWD,
               hr_mpix_per_s=lay.out_numel / 3 / (t_step * 1e-3) / 1e6)
    if name in ("C1", "C2"):
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            step()                                  # warm (one-time kernel setup) outside
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=st):
            step()
        row["step_graph_ms"] = median_ms(graph.replay, iters)
    if not quiet:
        print(json.dumps(row), flush=True)
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--configs", default="C1,C2,C3,C4,C5s,C5")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = [run(c, a.iters) for c in a.configs.split(",")]
    if a.out:
        Path(a.out).write_text(json.dumps({"device": torch.cuda.get_device_name(),
                                           "lib": gsr.version(), "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
