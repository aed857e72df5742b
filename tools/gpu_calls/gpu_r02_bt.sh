#!/bin/bash
# forward back list: single-half recurrences dispatched with one compare each
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5.py tests/test_gpu_limits.py -q -x --timeout 600 2>&1 | grep -E "^(FAILED|E )|passed|failed" | head -20
CFGS="C2 C4 C5s" timeout 1200 bash tools/ab_phase.sh 2>&1 | grep -E "==|C1|C2|C4|C5"
