timeout 300 python -m pytest tests/test_gpu_tc.py -q -x -k "gemm_cat" 2>&1 | tail -2
timeout 300 python tools/tools_pass_ab.py --configs c2,c4,c5 -
timeout 900 python -m pytest tests/test_gpu_unet_full.py tests/test_gpu_unet.py -q -x 2>&1 | tail -2
