#!/bin/bash
# GSR_BOUNDS_CHECK build (device asserts on the candidate-stream indices, staging slots and record
# positions) under the forward / binning GPU tests -- compute-sanitizer is closed on this pool
python __graft_entry__.py > /dev/null
GSR_LIB_PATH=tools/libgsr_E_bounds.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5.py tests/test_gpu_limits.py tests/test_gpu_formats.py tests/test_gpu_scale_vector.py tests/test_gpu_train.py -q --timeout 600 2>&1 | grep -E "^(FAILED|E )|passed|failed|assert" | head -20
GSR_LIB_PATH=tools/libgsr_E_bounds.so python tools/sanitize_run.py chunks 2>&1 | tail -1
GSR_LIB_PATH=tools/libgsr_E_bounds.so python -c "import paper_2501_06838_b200 as g; print(g._lib.load()._name)"
