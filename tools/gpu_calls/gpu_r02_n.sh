#!/bin/bash
# A/B of backward variants (merged blue-channel LDS; y-formulation) + backward parity
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5.py tests/test_gpu_train.py -q -x --timeout 600 2>&1 | tail -3
CFGS="C2 C4 C5s" timeout 900 bash tools/ab_run.sh 2>&1 | tail -20
