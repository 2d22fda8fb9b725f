ADX_LIB_VARIANT=tls python tools/tools_tc_timeline.py 2>&1 | grep "conv 48\|conv 12"
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -1
python tools/tools_pass_ab.py --configs c2,c4,c5 hd - hd -
