#!/bin/bash
python __graft_entry__.py > /dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_probe tools/mma_probe.cu && timeout 120 ./tools/mma_probe 2>&1 | tail -14
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu && timeout 300 ./tools/microbench > gpurun_out/r02_microbench.txt 2>&1; tail -20 gpurun_out/r02_microbench.txt
timeout 500 python -m pytest tests/test_gpu_dist.py -q -rf --timeout 200 > gpurun_out/pytest_dist.txt 2>&1; tail -4 gpurun_out/pytest_dist.txt | cut -c1-300
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 --deselect tests/test_gpu_dist.py > gpurun_out/pytest_gpu_r02e.txt 2>&1; tail -6 gpurun_out/pytest_gpu_r02e.txt | cut -c1-300
GSR_BENCH_SHARE_GPU=1 timeout 300 python bench.py --gpus 2 --images 2 --steps 2 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/bench_share2.json 2> gpurun_out/bench_share2.err; tail -2 gpurun_out/bench_share2.err; cut -c1-400 gpurun_out/bench_share2.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_render_(fwd2|bwd)" -c 2 -o gpurun_out/prof_r02e python tools/profile_run.py C5 4 > gpurun_out/ncu_r02e.log 2>&1; tail -2 gpurun_out/ncu_r02e.log
timeout 900 python tools/rank_projection.py --images 64 --iters 2 --out gpurun_out/r02_rank_projection.json 2>&1 | tail -6
