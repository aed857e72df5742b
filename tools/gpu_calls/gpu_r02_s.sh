#!/bin/bash
# full GPU suite + smoke + bench on the current tree
python __graft_entry__.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/pytest_gpu_r02s.txt 2>&1; tail -3 gpurun_out/pytest_gpu_r02s.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_r02s.json 2> gpurun_out/bench_r02s.err; tail -2 gpurun_out/bench_r02s.err; python -c "
import json; d=json.load(open('gpurun_out/bench_r02s.json')); r=d['roofline']
print(d['value'], d['ms_per_step'], d['e2e']['value'], r['frac'], r['other_kernel']['frac'], r['fwd_bwd_combined_frac'], d['phase_ms_per_step'])
for k,v in d['configs'].items(): print(k, v.get('fwd_ms'), v.get('bwd_ms'), v.get('step_ms'), v.get('step_graph_ms'))"
