python __graft_entry__.py > /dev/null
GSR_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --images 8 --steps 2 --warmup 3 2>&1 | tail -5
GSR_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --images 8 --steps 2 --warmup 3 --partition image 2>&1 | tail -3
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 2>&1 | tail -2
