#!/bin/bash
python __graft_entry__.py > /dev/null
timeout 120 python tools/dbg_k7.py 2>&1 | tail -5
timeout 500 python -m pytest tests/test_gpu_dist.py -q -x -rf --timeout 200 > gpurun_out/pytest_dist.txt 2>&1; tail -4 gpurun_out/pytest_dist.txt | cut -c1-300
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 --deselect tests/test_gpu_dist.py > gpurun_out/pytest_gpu_r02d.txt 2>&1; tail -6 gpurun_out/pytest_gpu_r02d.txt | cut -c1-300
timeout 300 python tools/bwd_gate_evidence.py gpurun_out/r02_bwd_gate.json 2>&1 | tail -6
CFGS="C2 C4 C5s" timeout 400 bash tools/ab_run.sh 2>&1 | tail -12
GSR_BENCH_SHARE_GPU=1 timeout 300 python bench.py --gpus 2 --images 2 --steps 2 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/bench_share2.json 2> gpurun_out/bench_share2.err; tail -2 gpurun_out/bench_share2.err; cut -c1-300 gpurun_out/bench_share2.json
timeout 600 python tools/rank_projection.py --images 16 --iters 2 2>&1 | tail -8
