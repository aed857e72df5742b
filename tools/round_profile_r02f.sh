#!/bin/bash
# Round-2 closing measurement (session 3, final HEAD after the alignment fix): GPU tests, smoke, the bench line (C5 + C1-C4), the reference arm,
# the ncu launch list of the bench command, the DRAM traffic of the two render kernels at the
# bench size, and ncu --set full captures of both kernels on a 4-image C5 slice and on C2.
python __graft_entry__.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/pytest_gpu_r02f.txt 2>&1; tail -2 gpurun_out/pytest_gpu_r02f.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02f.txt 2>&1; tail -1 gpurun_out/smoke_r02f.txt
timeout 900 python bench.py > gpurun_out/bench_r02f.json 2> gpurun_out/bench_r02f.err; tail -2 gpurun_out/bench_r02f.err; cut -c1-200 gpurun_out/bench_r02f.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r02f.json 2>&1; cut -c1-200 gpurun_out/bench_ref_r02f.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02f.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-configs > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_render_(fwd|bwd)" -s 2 -c 2 -o gpurun_out/traffic_r02f \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-configs > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_render_(fwd|bwd)" -c 2 \
    -o gpurun_out/prof_r02f_c5 python tools/profile_run.py C5 4 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_render_(fwd|bwd)" -c 2 \
    -o gpurun_out/prof_r02f_c2 python tools/profile_run.py C2 > /dev/null 2>&1
python tools/train_bench.py --out gpurun_out/train_bench_r02f.json > gpurun_out/train_bench_r02f.log 2>&1; tail -3 gpurun_out/train_bench_r02f.log
ls -la gpurun_out | tail -14
