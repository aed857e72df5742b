#!/bin/bash
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_train.py -q -rf --timeout 600 > gpurun_out/pytest_train.txt 2>&1; tail -4 gpurun_out/pytest_train.txt | cut -c1-300; grep -E "^E .*Assert" gpurun_out/pytest_train.txt | head -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/profile_run.py C2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python tools/profile_run.py C1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_render_(fwd2|bwd)" -c 2 -o gpurun_out/prof_c2 python tools/profile_run.py C2 > /dev/null 2>&1
ls gpurun_out | head -50
