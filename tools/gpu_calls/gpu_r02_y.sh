#!/bin/bash
python __graft_entry__.py > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_render_(fwd2|bwd)" -c 2 -o gpurun_out/prof_r02y_c5 python tools/profile_run.py C5 4 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_render_(fwd2|bwd)" -c 2 -o gpurun_out/prof_r02y_c2 python tools/profile_run.py C2 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep | tail -3
