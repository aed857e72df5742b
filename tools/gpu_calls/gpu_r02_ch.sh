#!/bin/bash
# A/B: small forward tiles with a 6-CTA register budget (80 registers, small spills)
python __graft_entry__.py > /dev/null
CFGS="C1 C2" timeout 1200 bash tools/ab_phase.sh 2>&1 | grep -E "==|C1|C2|C4|C5"
