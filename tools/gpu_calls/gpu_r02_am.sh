#!/bin/bash
python __graft_entry__.py > /dev/null
timeout 600 ncu --set full --clock-control none -k regex:"k_keys|k_records" -c 2 -o gpurun_out/prof_keys python tools/profile_run.py C5 4 > /dev/null 2>&1
ls -la gpurun_out/prof_keys*
