#!/bin/bash
# small-config forward 1x8 px per lane (32x8 tiles, column halves) vs 1x4 (16x8); parity
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_train.py tests/test_gpu_scale_vector.py tests/test_gpu_formats.py tests/test_gpu_graph.py -q -x --timeout 600 2>&1 | tail -3
CFGS="C1 C2 C4" timeout 900 bash tools/ab_run.sh 2>&1 | tail -12
