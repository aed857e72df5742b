#!/bin/bash
# forward warp buffers per configuration (large 96, small 48), epilogue aliasing the records
python __graft_entry__.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | grep -E "^(FAILED|E )|passed|failed" | head -20
python tools/phase_time.py C1 C2 C4 C5s 2>&1 | tail -4
