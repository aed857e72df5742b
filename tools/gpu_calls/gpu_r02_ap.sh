#!/bin/bash
python __graft_entry__.py > /dev/null
CFGS="C1 C2 C5s" timeout 1200 bash tools/ab_phase.sh 2>&1 | grep -E "==|C1|C2|C5"
