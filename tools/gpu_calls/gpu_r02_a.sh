#!/bin/bash
# round-2 GPU session A: full GPU test suite + backward gate evidence
python __graft_entry__.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/pytest_gpu_r02a.txt 2>&1; tail -5 gpurun_out/pytest_gpu_r02a.txt
timeout 600 python tools/bwd_gate_evidence.py gpurun_out/r02_bwd_gate.json 2>&1 | tail -8
