#!/bin/bash
# forward back list on running 32-bit shared addresses
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5.py tests/test_gpu_limits.py tests/test_gpu_formats.py -q -x --timeout 600 2>&1 | grep -E "^(FAILED|E )|passed|failed" | head -20
python tools/phase_time.py C1 C2 C4 C5s 2>&1 | tail -4
python tools/phase_time.py C1 C2 C4 C5s 2>&1 | tail -4
