#!/bin/bash
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_streamed.py -q --timeout 600 2>&1 | grep -vE "^frame #" | tail -40
