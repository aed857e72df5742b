python __graft_entry__.py > /dev/null
CFGS="C2 C3 C4 C5s" timeout 900 bash tools/ab_run.sh 2>&1 | tee gpurun_out/ab47.txt
GSR_LIB_PATH=tools/libgsr_E37med.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fwd" 2>&1 | tail -2
