#!/bin/bash
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5.py tests/test_gpu_limits.py tests/test_gpu_formats.py tests/test_gpu_train.py -q -x --timeout 600 2>&1 | grep -E "^(FAILED|E )|Error|assert|passed|failed" | head -40
