#!/bin/bash
# backward: reach-trimmed cell rows from the CandStream table, walked row by row: parity + A/B
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5.py tests/test_gpu_limits.py tests/test_gpu_train.py -q -x --timeout 600 2>&1 | grep -E "^(FAILED|E )|Error|passed|failed" | head -20
CFGS="C1 C2 C4 C5s" timeout 1200 bash tools/ab_phase.sh 2>&1 | grep -E "==|C1|C2|C4|C5"
