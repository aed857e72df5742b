#!/bin/bash
python __graft_entry__.py > /dev/null
timeout 120 python tools/dbg_k7.py 2>&1 | tail -8
timeout 400 python -m pytest tests/test_gpu_dist.py -q -x -rf --timeout 200 -p no:cacheprovider > gpurun_out/pytest_dist.txt 2>&1; tail -30 gpurun_out/pytest_dist.txt | cut -c1-300
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5.py tests/test_gpu_scale_vector.py tests/test_gpu_formats.py tests/test_gpu_train.py tests/test_gpu_limits.py tests/test_gpu_graph.py -q -rf --timeout 300 > gpurun_out/pytest_fwd3.txt 2>&1; tail -6 gpurun_out/pytest_fwd3.txt
timeout 300 python tools/quick_time.py C1 C2 C4 C5s 2>&1 | tail -5
