#!/bin/bash
# Round-2 evidence (run on the GPU box via gpurun; outputs in gpurun_out/): bench lines (c2 with the
# CPU baseline and the f32 parity line, c4, c5, the reference arm), the ncu launch list of the bench
# command, the DRAM traffic of one c2 pass per kernel family, and one ncu --set full capture of the
# level-0 conv and self-attention.
set -x
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err
python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_c2_reference.json 2> gpurun_out/r02_ref.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity-line > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -c 3000 --csv \
    --log-file gpurun_out/r02_c2_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity-line \
    > gpurun_out/r02_ncu_bench.log 2>&1
python tools/tools_launch_agg.py gpurun_out/r02_c2_launches.csv 4 > gpurun_out/r02_c2_launch_agg.txt
python tools/tools_unet_pass.py > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r02_c2_dram_traffic_ncu.csv python tools/tools_unet_pass.py > gpurun_out/r02_ncu_traffic.log 2>&1
python tools/tools_ncu_traffic.py gpurun_out/r02_c2_dram_traffic_ncu.csv 4 > gpurun_out/r02_c2_dram_traffic.json
python tools/tools_unet_layer0.py > gpurun_out/plain3.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"tc_gemm_kernel|attn_kernel" -c 2 \
    -o gpurun_out/r02_layer0 python tools/tools_unet_layer0.py > gpurun_out/r02_ncu_full.log 2>&1
python tools/tools_ncu_summary.py gpurun_out/r02_layer0.ncu-rep > gpurun_out/r02_layer0_ncu_full_summary.txt
python tools/tools_sol.py c2 bf16 > gpurun_out/r02_c2_sol_bf16.txt 2>&1
python tools/tools_sol.py c2 f32 > gpurun_out/r02_c2_sol_f32.txt 2>&1
python tools/tools_shape_profile.py c2 bf16 > gpurun_out/r02_c2_shape_profile.txt 2>&1
