#!/bin/bash
python __graft_entry__.py > /dev/null
timeout 500 python -m pytest tests/test_gpu_dist.py -q -rf --timeout 200 > gpurun_out/pytest_dist.txt 2>&1; tail -3 gpurun_out/pytest_dist.txt | cut -c1-300
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 --deselect tests/test_gpu_dist.py > gpurun_out/pytest_gpu_r02g.txt 2>&1; tail -4 gpurun_out/pytest_gpu_r02g.txt | cut -c1-300
CFGS="C4 C5s" timeout 600 bash tools/ab_run.sh 2>&1 | tail -12
