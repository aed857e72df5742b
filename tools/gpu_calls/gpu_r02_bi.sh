#!/bin/bash
# forward candidate stream + cell reach (cleaned build): full GPU suite, smoke, phases
python __graft_entry__.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | grep -E "^(FAILED|E )|passed|failed" | head -20
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python tools/phase_time.py C1 C2 C4 C5s 2>&1 | tail -4
