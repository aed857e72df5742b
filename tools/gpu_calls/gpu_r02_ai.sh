#!/bin/bash
# compute-sanitizer on the closing kernels (racecheck / synccheck / memcheck)
python __graft_entry__.py > /dev/null
mkdir -p gpurun_out/san2
for t in racecheck synccheck memcheck; do for c in C1 C2 C5band subset; do
  timeout 900 compute-sanitizer --tool $t --kernel-name kns=k_ --print-limit 20 python tools/sanitize_run.py $c > gpurun_out/san2/san_${t}_${c}.txt 2>&1; echo "$t $c: $(grep -E 'SUMMARY|ok' gpurun_out/san2/san_${t}_${c}.txt | tr '\n' ' ')"
done; done
