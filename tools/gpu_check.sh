timeout 600 python -m pytest tests/test_gpu_tc.py -q -x -k "geglu or stride2 or gemm_cat" 2>&1 | tail -3
