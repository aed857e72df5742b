#!/bin/bash
# per-rank projection (rank r of G on one B200) with the session-3 kernels; 2-rank CUDA band test
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x --timeout 600 2>&1 | tail -2
timeout 1500 python tools/rank_projection.py --images 64 --iters 2 --out gpurun_out/r02_rank_projection_final.json 2>&1 | grep -E "G=|plain"
