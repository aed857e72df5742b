"""NEXT-2: the paper's data-parallel training layout for the rasterizer step
(batch 64 on 4 GPUs = 16 LR patches of 48x48 per GPU, s ~ U[1, 4] per patch, m = 16),
one process per GPU through the same launcher as bench.py.

Each rank runs the fused training step (activations -> render -> L1 loss -> raw gradients,
ops.train_step_l1, replayed from a CUDA graph: ops.TrainStepGraph) on ITS OWN 16 patches -- the
rasterizer has no cross-sample coupling, so data parallelism needs no exchange inside the step;
the raw gradients flow back into each rank's copy of the network, whose own gradients the
training framework all-reduces (outside this library). The only collective here is the global
mean loss (an all-reduce of one float64), as a training loop would log it. The L1 gradient is
normalised by the GLOBAL element count (inv_numel), so the per-rank gradients are those of the
global mean loss.

Timing: W warm-up steps, then K steps bracketed by barrier + synchronize, max over ranks.
usage: python tools/train_dp.py --gpus 4 [--steps 50] [--warmup 5] [--patches 16] [--lr 48]
       [--smax 4]        (GSR_BENCH_SHARE_GPU=1: every rank on cuda:0 over gloo, functional only)"""
import argparse
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=4)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--patches", type=int, default=16)
    ap.add_argument("--lr", type=int, default=48)
    ap.add_argument("--smax", type=float, default=4.0)
    a = ap.parse_args()
    share = os.environ.get("GSR_BENCH_SHARE_GPU") == "1"
    if "WORLD_SIZE" not in os.environ and a.gpus > 1:
        import torch
        if a.gpus > torch.cuda.device_count() and not share:
            raise SystemExit(f"--gpus {a.gpus}: only {torch.cuda.device_count()} GPU(s) visible")
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        return subprocess.call([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                f"--nproc-per-node={a.gpus}", "--master-addr=127.0.0.1",
                                f"--master-port={port}", str(Path(__file__).resolve()),
                                *sys.argv[1:]])
    import torch
    import torch.distributed as dist
    import gsr_synth as S
    import paper_2501_06838_b200 as gsr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if share else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("gloo" if share else "nccl",
                                **({} if share else {"device_id": dev}))
    # this rank's batch: its own patches and per-patch scales (seeded by rank)
    B, P, M = a.patches, a.lr, 16
    rng = np.random.default_rng(100 + rank)
    scales = rng.uniform(1.0, a.smax, B)
    n1 = M * P * P
    ref = np.concatenate([S.reference_grid(P, P, M) for _ in range(B)]).astype(np.float32)
    n = B * n1
    raw = dict(raw_alpha=rng.normal(-3, 1, n), offset=rng.uniform(-0.5, 0.5, (n, 2)),
               raw_sigma=rng.normal(-0.5, 0.5, (n, 2)), raw_rho=rng.normal(0, 0.5, n),
               raw_color=rng.normal(0, 1, (n, 3)))
    args = [torch.from_numpy(raw[k].astype(np.float32)).to(dev) if k != "ref" else
            torch.from_numpy(ref).to(dev)
            for k in ("raw_alpha", "offset", "ref", "raw_sigma", "raw_rho", "raw_color")]
    lay = gsr.layout([gsr.Image(P, P, float(s), k * n1, n1) for k, s in enumerate(scales)])
    gt = torch.rand(lay.out_numel, device=dev, generator=torch.Generator(device=dev)
                    .manual_seed(200 + rank))
    # global element count: every rank's gradient is that of the global mean loss
    tot = torch.tensor([float(lay.out_numel)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot)
    step = gsr.TrainStepGraph(lay, n, ratio=0.1, inv_numel=1.0 / float(tot.item()), device=dev)

    def one():
        out, loss, grads = step(*args, gt)
        if world > 1:
            lsum = loss.clone()
            dist.all_reduce(lsum)            # global mean loss (sum of the rank partial means)
            return lsum
        return loss

    for _ in range(a.warmup):
        one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        gl = one()
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1) / a.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    if rank == 0:
        print(json.dumps({"workload": f"{B} x {P}x{P} LR patches per rank, s ~ U[1,{a.smax:g}], "
                                      f"m = 16 (P:1708-1709)",
                          "ranks": world, "global_batch": B * world,
                          "ms_per_step": ms, "patches_per_s": B * world / (ms * 1e-3),
                          "hr_mpix_per_s": lay.out_numel / 3 * world / (ms * 1e-3) / 1e6,
                          "global_mean_loss": float(gl.item()),
                          "functional_only_shared_gpu": share,
                          "lib": gsr.version()}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
