#!/bin/bash
python __graft_entry__.py > /dev/null
for g in 16 32 64; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-configs --no-cpu-baseline --e2e-groups $g 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($g, d['value'], d['e2e'])"
done
