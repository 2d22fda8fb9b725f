python tools/tools_unet_layer0.py > gpurun_out/p1.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"attn_kernel" -c 1 \
    -o gpurun_out/r02_attn_sk python tools/tools_unet_layer0.py > gpurun_out/ncu_sk.log 2>&1
python tools/tools_ncu_summary.py gpurun_out/r02_attn_sk.ncu-rep > gpurun_out/r02_attn_sk_ncu_full_summary.txt
python tools/tools_attn_f32_one.py > gpurun_out/p2.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"attn_kernel" -c 1 \
    -o gpurun_out/r02_attn_f32 python tools/tools_attn_f32_one.py > gpurun_out/ncu_f32.log 2>&1
python tools/tools_ncu_summary.py gpurun_out/r02_attn_f32.ncu-rep > gpurun_out/r02_attn_f32_ncu_full_summary.txt
