#!/bin/bash
# Run on the GPU box (gpurun): the bench line, the ncu launch list of the same bench command,
# and one ncu --set full capture of the level-0 conv and self-attention; outputs in gpurun_out/.
set -x
python bench.py > gpurun_out/prof_bench_c2.json 2> gpurun_out/prof_bench_c2.err
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -c 3000 --csv \
    --log-file gpurun_out/prof_c2_launches.csv python bench.py --steps 1 --warmup 3 > gpurun_out/prof_ncu_bench.log 2>&1
python tools/tools_launch_agg.py gpurun_out/prof_c2_launches.csv 4 > gpurun_out/prof_c2_launch_agg.txt
python tools/tools_launch_shapes.py gpurun_out/prof_c2_launches.csv 4 > gpurun_out/prof_c2_launch_shapes.txt
ncu --set full --import-source on --clock-control none -k regex:"tc_gemm_kernel|attn_kernel" -c 2 \
    -o gpurun_out/prof_layer0 python tools/tools_unet_layer0.py > gpurun_out/prof_ncu_full.log 2>&1
python tools/tools_ncu_summary.py gpurun_out/prof_layer0.ncu-rep > gpurun_out/prof_layer0_summary.txt
python tools/tools_shape_profile.py c2 > gpurun_out/prof_c2_shapes.txt 2>&1
