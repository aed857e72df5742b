#!/bin/bash
# backward: w += 2D inside unrolled column blocks (re-anchored per block): GPU suite + A/B vs HEAD
python __graft_entry__.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | grep -E "^(FAILED|E )|passed|failed" | head -20
CFGS="C1 C2 C4 C5s" timeout 1200 bash tools/ab_phase.sh 2>&1 | grep -E "==|C1|C2|C4|C5"
python tools/bwd_gate_evidence.py 2>&1 | tail -8
