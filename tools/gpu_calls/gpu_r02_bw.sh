#!/bin/bash
# forward front loop on one 32-bit shared address (67 instructions per Gaussian)
python __graft_entry__.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | grep -E "^(FAILED|E )|passed|failed" | head -20
python tools/phase_time.py C1 C2 C4 C5s 2>&1 | tail -4
python tools/phase_time.py C1 C2 C4 C5s 2>&1 | tail -4
