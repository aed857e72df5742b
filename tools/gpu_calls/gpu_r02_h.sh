#!/bin/bash
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_dist.py -q -rf --timeout 600 > gpurun_out/pytest_train.txt 2>&1; tail -4 gpurun_out/pytest_train.txt | cut -c1-300
timeout 900 python tools/rank_projection.py --images 64 --iters 2 --out gpurun_out/r02_rank_projection.json 2>&1 | tail -6
for t in racecheck synccheck; do for c in C1 C2 C5band subset; do
  timeout 600 compute-sanitizer --tool $t --kernel-name kns=k_ --print-limit 20 python tools/sanitize_run.py $c > gpurun_out/san_${t}_${c}.txt 2>&1; echo "$t $c: $(tail -1 gpurun_out/san_${t}_${c}.txt)"
done; done
