for v in sk4 - sk4 -; do if [ "$v" = "-" ]; then unset ADX_LIB_VARIANT; else export ADX_LIB_VARIANT=$v; fi; echo "== $v"; python tools/tools_attn_bench.py 2>/dev/null | head -1; done
ADX_LIB_VARIANT=sk4 timeout 300 python -m pytest tests/test_gpu_tc.py -q -x -k "attention and not f32 and not temporal" 2>&1 | tail -1
