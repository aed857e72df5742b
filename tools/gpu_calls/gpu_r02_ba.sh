#!/bin/bash
# Session-3 start: HEAD (per-block support extents in K1) -- full GPU tests, smoke, bench line, phases.
python __graft_entry__.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/pytest_gpu_ba.txt 2>&1; tail -3 gpurun_out/pytest_gpu_ba.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_ba.json 2> gpurun_out/bench_ba.err; tail -2 gpurun_out/bench_ba.err; cut -c1-400 gpurun_out/bench_ba.json
python tools/phase_time.py C1 C2 C4 C5s 2>&1 | tail -6
