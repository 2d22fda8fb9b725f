timeout 300 python -m pytest tests/test_gpu_tc.py -q -x -k "deterministic" 2>&1 | tail -2
