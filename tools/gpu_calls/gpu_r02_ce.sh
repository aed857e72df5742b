#!/bin/bash
# A/B: 4 warps per large forward tile with the candidate stream
python __graft_entry__.py > /dev/null
CFGS="C4 C5s" timeout 1200 bash tools/ab_phase.sh 2>&1 | grep -E "==|C1|C2|C4|C5"
