#!/bin/bash
# A/B of the fused attention kernels (ADX_ATTN_V=1: round-1 kernel, default v2) at the UNet shapes
for v in 1 2; do echo "== v$v"; ADX_ATTN_V=$v python tools/tools_attn_bench.py; done
