#!/bin/bash
python __graft_entry__.py > /dev/null
CFGS="C2 C4 C5s" timeout 600 bash tools/ab_run.sh 2>&1 | tail -16
GSR_BENCH_SHARE_GPU=1 timeout 300 python tools/train_dp.py --gpus 2 --steps 10 2>&1 | tail -2
timeout 300 python tools/train_dp.py --gpus 1 --steps 30 2>&1 | tail -1
