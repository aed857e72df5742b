#!/bin/bash
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -q -x --timeout 600 -k "self_launch or train_dp or order_invariance" 2>&1 | tail -4
