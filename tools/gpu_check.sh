timeout 300 python -m pytest tests/test_gpu_tc.py -q -x -k "attention" 2>&1 | tail -1
for sk in 0 1; do ADX_ATTN_SK=$sk python tools/tools_attn_bench.py | head -3; done
