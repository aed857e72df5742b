#!/bin/bash
# forward record prefetch (one Gaussian ahead) A/B, small and large configuration
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5.py -q -x --timeout 600 2>&1 | tail -2
CFGS="C1 C2 C4 C5s" timeout 1200 bash tools/ab_run.sh 2>&1 | tail -22
