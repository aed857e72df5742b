#!/bin/bash
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -k "tile_lists" 2>&1 | tail -2
