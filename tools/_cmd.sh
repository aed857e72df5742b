python __graft_entry__.py > /dev/null
CFGS="C2 C3 C4 C5s" timeout 900 bash tools/ab_run.sh 2>&1 | tee gpurun_out/ab45.txt
