python __graft_entry__.py > /dev/null
python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu22.txt 2>&1; tail -5 gpurun_out/pytest_gpu22.txt
python tools/quick_time.py C1 C2 C3 C4 C5s 2>&1 | tee gpurun_out/q22.txt
