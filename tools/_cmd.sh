python __graft_entry__.py > /dev/null
python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu30.txt 2>&1; tail -3 gpurun_out/pytest_gpu30.txt
CFGS="C1 C2 C3 C4 C5s" bash tools/ab_run.sh 2>&1 | tee gpurun_out/ab30.txt
python bench.py > gpurun_out/bench30.json 2> gpurun_out/bench30.err; tail -2 gpurun_out/bench30.err; cat gpurun_out/bench30.json
