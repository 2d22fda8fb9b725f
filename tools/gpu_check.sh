set -x
timeout 300 python -m pytest tests/test_gpu_tc.py -q -x -k "f32" 2>&1 | tail -5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r02_c2_f32_fused_launches.csv python tools/tools_unet_pass.py c2 f32 > /dev/null 2>&1
python tools/tools_launch_agg.py gpurun_out/r02_c2_f32_fused_launches.csv 2>&1 | head -30
