python __graft_entry__.py > /dev/null
timeout 600 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu43.txt 2>&1; tail -3 gpurun_out/pytest_gpu43.txt
CFGS="C1 C2 C3 C4 C5s" timeout 900 bash tools/ab_run.sh 2>&1 | tee gpurun_out/ab43.txt
