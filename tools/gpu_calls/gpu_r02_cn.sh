#!/bin/bash
# data-parallel training launcher with the closing kernels (1 rank; 2 and 4 ranks sharing the GPU)
python __graft_entry__.py > /dev/null
timeout 300 python tools/train_dp.py --gpus 1 --steps 30 2>&1 | tail -1 > gpurun_out/r02_train_dp1_final.json
GSR_BENCH_SHARE_GPU=1 timeout 300 python tools/train_dp.py --gpus 2 --steps 10 2>&1 | tail -1 > gpurun_out/r02_train_dp2_shared_final.json
GSR_BENCH_SHARE_GPU=1 timeout 300 python tools/train_dp.py --gpus 4 --steps 10 2>&1 | tail -1 > gpurun_out/r02_train_dp4_shared_final.json
cat gpurun_out/r02_train_dp*_final.json | cut -c1-300
