#!/bin/bash
python __graft_entry__.py > /dev/null
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_c5.py tests/test_gpu_parity.py tests/test_gpu_scale_vector.py -m gpu -q -rf --timeout 900 > gpurun_out/pytest_gpu_r02b.txt 2>&1; tail -5 gpurun_out/pytest_gpu_r02b.txt
timeout 600 python tools/bwd_gate_evidence.py gpurun_out/r02_bwd_gate.json 2>&1 | tail -8
GSR_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --images 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_share2.json 2> gpurun_out/bench_share2.err; tail -3 gpurun_out/bench_share2.err; cut -c1-400 gpurun_out/bench_share2.json
