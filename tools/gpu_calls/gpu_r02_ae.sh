#!/bin/bash
python __graft_entry__.py > /dev/null
timeout 1500 python tools/rank_projection.py --images 64 --iters 2 --out gpurun_out/r02_rank_projection.json 2>&1 | tail -12
GSR_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --images 4 --steps 2 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/bench_share2.json 2> gpurun_out/bench_share2.err; tail -2 gpurun_out/bench_share2.err; cut -c1-300 gpurun_out/bench_share2.json
