#!/bin/bash
# forward tile lists materialised (gsr_debug_fwd_tile_lists) + full GPU suite + phase check
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -k "fwd_tile_lists" 2>&1 | grep -E "^(FAILED|E )|passed|failed|Error" | head -20
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | grep -E "^(FAILED|E )|passed|failed" | head -10
python tools/phase_time.py C2 C4 C5s 2>&1 | tail -3
