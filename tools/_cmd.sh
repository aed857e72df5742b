python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_c5.py -q -rf -s 2>&1 | tail -8
