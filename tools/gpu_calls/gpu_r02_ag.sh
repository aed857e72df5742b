#!/bin/bash
python __graft_entry__.py > /dev/null
for i in 1 2; do
CFGS="C4 C5s" timeout 1200 bash tools/ab_phase.sh 2>&1 | grep -E "==|C4|C5"
done
