#!/bin/bash
# time the attention kernel in each library variant given (ADX_LIB_VARIANT), v1 and v2
for var in "$@"; do for v in 1 2; do echo "== $var v$v"; ADX_LIB_VARIANT=$var ADX_ATTN_V=$v python tools/tools_attn_bench.py 2>&1 | head -3; done; done
