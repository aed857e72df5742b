#!/bin/bash
# streamed host-memory step with ramped image groups (1-image first / last group): test + e2e bench
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_streamed.py -q --timeout 600 2>&1 | tail -2
timeout 900 python bench.py --no-cpu-baseline --no-configs > gpurun_out/bench_ck.json 2> gpurun_out/bench_ck.err; python -c "
import json;d=json.loads(open('gpurun_out/bench_ck.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'])"
