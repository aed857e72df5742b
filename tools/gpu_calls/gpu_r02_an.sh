#!/bin/bash
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5.py tests/test_gpu_limits.py tests/test_gpu_formats.py -q -x --timeout 600 2>&1 | tail -2
python tools/phase_time.py C1 C2 C4 C5s 2>&1 | tail -4
timeout 600 ncu --set full --clock-control none -k regex:"k_keys|k_records" -c 2 -o gpurun_out/prof_keys2 python tools/profile_run.py C5 4 > /dev/null 2>&1
