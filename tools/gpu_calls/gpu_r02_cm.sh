#!/bin/bash
# misaligned output buffers (float4 epilogue checks absolute alignment) + streamed ramped groups + e2e
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_streamed.py tests/test_gpu_parity.py -q --timeout 600 -k "streamed or any_float_offset" 2>&1 | grep -vE "^frame #" | tail -3
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | grep -E "^(FAILED|E )|passed|failed" | head -10
timeout 900 python bench.py --no-cpu-baseline --no-configs > gpurun_out/bench_cm.json 2> gpurun_out/bench_cm.err; python -c "
import json;d=json.loads(open('gpurun_out/bench_cm.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['fwd_bwd_combined_frac'])"
