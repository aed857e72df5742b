#!/bin/bash
python __graft_entry__.py > /dev/null
for i in 1 2; do CFGS="C1 C2" timeout 1200 bash tools/ab_phase.sh 2>&1 | grep -E "==|C1|C2"; done
