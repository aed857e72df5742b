#!/bin/bash
# Source-level ncu capture of the forward (C5 slice, C2) and backward (C5 slice): stall samples per loop
python __graft_entry__.py > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_render_(fwd|bwd)" -c 2 \
    -o gpurun_out/prof_bb_c5 python tools/profile_run.py C5 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_render_fwd" -c 1 \
    -o gpurun_out/prof_bb_c2 python tools/profile_run.py C2 > /dev/null 2>&1
ls -la gpurun_out/
