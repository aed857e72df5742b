#!/bin/bash
# pipe-rate microbenchmark (profiles/r02_microbench.txt, DESIGN 7) + A/B: forward scan depth 3, backward unroll 4
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/microbench tools/microbench.cu && /tmp/microbench > gpurun_out/r02_microbench.txt 2>&1; tail -5 gpurun_out/r02_microbench.txt
python __graft_entry__.py > /dev/null
CFGS="C1 C2 C4 C5s" timeout 1200 bash tools/ab_phase.sh 2>&1 | grep -E "==|C1|C2|C4|C5"
