#!/bin/bash
# NEXT-3 sweeps with the session-3 kernels
python __graft_entry__.py > /dev/null
timeout 1200 python tools/sweep.py --out gpurun_out/r02_sweep.json 2>&1 | tail -30
ls gpurun_out/ | grep sweep
