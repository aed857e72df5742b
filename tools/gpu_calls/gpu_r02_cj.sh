#!/bin/bash
# GSR_BOUNDS_CHECK build (device asserts: forward candidate stream / staging, radix scatter
# positions, cell-reach keys) under the whole GPU suite
python __graft_entry__.py > /dev/null
GSR_LIB_PATH=tools/libgsr_E_bounds.so timeout 1800 python -m pytest tests -m gpu -q --timeout 600 2>&1 | grep -E "^(FAILED|E )|passed|failed" | head -20
GSR_LIB_PATH=tools/libgsr_E_bounds.so python tools/sanitize_run.py chunks 2>&1 | tail -1
GSR_LIB_PATH=tools/libgsr_E_bounds.so python tools/sanitize_run.py subset 2>&1 | tail -1
