#!/bin/bash
# compute-sanitizer on the session-3 kernels (candidate stream, cell reach, mask words, radix)
python __graft_entry__.py > /dev/null
mkdir -p gpurun_out/san3
for t in racecheck synccheck memcheck; do for c in C1 C2 C5band subset chunks; do
  timeout 900 compute-sanitizer --tool $t --kernel-name kns=k_ --print-limit 20 python tools/sanitize_run.py $c > gpurun_out/san3/san_${t}_${c}.txt 2>&1; echo "$t $c: $(grep -E 'SUMMARY|ok' gpurun_out/san3/san_${t}_${c}.txt | tr '\n' ' ')"
done; done
