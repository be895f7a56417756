timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "bfs" 2>&1 | tail -3
