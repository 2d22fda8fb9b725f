timeout 300 python -m pytest tests/test_gpu_tc.py -q -x -k "attention and not f32 and not temporal" 2>&1 | tail -1
ADX_ATTN_SK=1 timeout 300 python -m pytest tests/test_gpu_tc.py -q -x -k "attention and not f32 and not temporal" 2>&1 | tail -1
for sk in 0 1; do echo "== SK=$sk"; ADX_ATTN_SK=$sk python tools/tools_attn_bench.py; done
