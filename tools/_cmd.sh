python __graft_entry__.py > /dev/null
timeout 600 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu44.txt 2>&1; tail -3 gpurun_out/pytest_gpu44.txt
timeout 300 python tools/quick_time.py C1 C2 C3 C4 C5s 2>&1 | tee gpurun_out/q44.txt
timeout 600 python tools/train_bench.py --out gpurun_out/train_bench44.json 2>&1 | tail -4
