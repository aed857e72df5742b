python __graft_entry__.py > /dev/null
python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu26.txt 2>&1; tail -3 gpurun_out/pytest_gpu26.txt
python tools/quick_time.py C1 C2 C3 C4 C5s 2>&1 | tee gpurun_out/q26.txt
echo "== strided"; GSR_LIB_PATH=tools/libgsr_E1strided.so python tools/quick_time.py C1 C2 C3 C4 C5s 2>&1
