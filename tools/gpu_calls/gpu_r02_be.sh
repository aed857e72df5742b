#!/bin/bash
# C4 forward: source-level ncu of the old producer vs the candidate stream (both without reach)
python __graft_entry__.py > /dev/null
for v in noreach vs_noreach; do
GSR_LIB_PATH=tools/libgsr_E_$v.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_render_fwd" -c 1 \
    -o gpurun_out/prof_be_c4_$v python tools/profile_run.py C4 > /dev/null 2>&1
done
ls gpurun_out
