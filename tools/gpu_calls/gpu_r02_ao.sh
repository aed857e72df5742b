#!/bin/bash
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5.py -q -x --timeout 600 2>&1 | tail -2
for i in 1 2 3; do python tools/phase_time.py C1 C2 2>&1 | tail -2; done
