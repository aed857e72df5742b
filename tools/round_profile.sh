#!/bin/bash
# One GPU session: parity tests, the bench line, the ncu launch list of the bench command and one
# ncu --set full capture of the two render kernels on the bench workload. Outputs in gpurun_out/.
set -x
python __graft_entry__.py
python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_full.txt 2>&1; tail -3 gpurun_out/pytest_gpu_full.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_under_ncu.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_render_(fwd|bwd)" -s 2 -c 2 \
    -o gpurun_out/prof_bench python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
ls -la gpurun_out
