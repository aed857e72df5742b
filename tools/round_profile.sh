#!/bin/bash
# One GPU session: parity tests, smoke, the bench line (C5), the ncu launch list of the bench
# command, a DRAM-traffic capture of the two render kernels at the bench size, and an
# ncu --set full capture of both kernels on a 4-image slice. Outputs in gpurun_out/.
set -x
python __graft_entry__.py
python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_full.txt 2>&1; tail -3 gpurun_out/pytest_gpu_full.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_under_ncu.json 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_render_(fwd|bwd)" -s 2 -c 2 -o gpurun_out/traffic \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_render_(fwd|bwd)" -c 2 \
    -o gpurun_out/prof_c5x4 python tools/profile_run.py C5 4 > gpurun_out/ncu_c5x4.log 2>&1
ls -la gpurun_out
