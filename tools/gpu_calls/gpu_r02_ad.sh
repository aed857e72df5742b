#!/bin/bash
python __graft_entry__.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_ad.txt 2>&1; tail -2 gpurun_out/pytest_ad.txt
python tools/phase_time.py C1 C2 C4 C5s 2>&1 | tail -4
