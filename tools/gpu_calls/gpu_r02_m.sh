#!/bin/bash
# round-2 session B: small-problem evidence (C1/C2 launch lists + ncu full of the C2 render
# kernels), compute-sanitizer logs, the data-parallel training launcher at 1 GPU and 2 shared ranks
python __graft_entry__.py > /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/profile_run.py C2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python tools/profile_run.py C1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_render_(fwd2|bwd)" -c 2 -o gpurun_out/prof_c2 python tools/profile_run.py C2 > /dev/null 2>&1
for t in racecheck synccheck memcheck; do for c in C1 C2 C5band subset; do
  timeout 900 compute-sanitizer --tool $t --kernel-name kns=k_ --print-limit 20 python tools/sanitize_run.py $c > gpurun_out/san_${t}_${c}.txt 2>&1; echo "$t $c: $(grep -E 'ERROR SUMMARY|ok' gpurun_out/san_${t}_${c}.txt | tr '\n' ' ')"
done; done
timeout 300 python tools/train_dp.py --gpus 1 --steps 50 > gpurun_out/train_dp1.json 2> gpurun_out/train_dp1.err; tail -1 gpurun_out/train_dp1.json
GSR_BENCH_SHARE_GPU=1 timeout 300 python tools/train_dp.py --gpus 2 --steps 10 > gpurun_out/train_dp2_shared.json 2> gpurun_out/train_dp2_shared.err; tail -1 gpurun_out/train_dp2_shared.json
GSR_BENCH_SHARE_GPU=1 timeout 300 python tools/train_dp.py --gpus 4 --steps 10 > gpurun_out/train_dp4_shared.json 2> gpurun_out/train_dp4_shared.err; tail -1 gpurun_out/train_dp4_shared.json
ls gpurun_out | head -60
