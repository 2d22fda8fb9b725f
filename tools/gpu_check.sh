ADX_TC_TRACE=1 python tools/tools_unet_pass.py c2 2>&1 | grep "M=144 N=10240"
timeout 300 python -m pytest tests/test_gpu_tc.py -q -x -k "geglu" 2>&1 | tail -1
python tools/tools_pass_ab.py --configs c2 - - -
