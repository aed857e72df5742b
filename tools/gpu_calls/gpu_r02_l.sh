#!/bin/bash
python __graft_entry__.py > /dev/null
CFGS="C1 C2 C4" timeout 600 bash tools/ab_run.sh 2>&1 | tail -16
