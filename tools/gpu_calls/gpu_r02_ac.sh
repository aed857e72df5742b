#!/bin/bash
python __graft_entry__.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2
CFGS="C1 C2 C3 C4 C5s" timeout 1200 bash tools/ab_phase.sh 2>&1 | tail -15
