#!/bin/bash
python __graft_entry__.py > /dev/null
CFGS="C2 C4 C5s" timeout 1200 bash tools/ab_phase.sh 2>&1 | tail -16
