#!/bin/bash
# forward: lane-level interleave over the split-K cluster, window masks as tile bit masks (small
# tiles): GPU suite + A/B vs HEAD, C2 source-level ncu
python __graft_entry__.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | grep -E "^(FAILED|E )|passed|failed" | head -20
CFGS="C1 C2 C4 C5s" timeout 1200 bash tools/ab_phase.sh 2>&1 | grep -E "==|C1|C2|C4|C5"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_render_fwd" -c 1 \
    -o gpurun_out/prof_bl_c2 python tools/profile_run.py C2 > /dev/null 2>&1
