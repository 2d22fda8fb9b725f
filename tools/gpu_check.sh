python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err
python tools/tools_sol.py c2 bf16 > gpurun_out/r02_c2_sol_bf16.txt 2>&1
python tools/tools_shape_profile.py c2 bf16 > gpurun_out/r02_c2_shape_profile.txt 2>&1
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity-line > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -c 3000 --csv \
    --log-file gpurun_out/r02_c2_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity-line \
    > gpurun_out/r02_ncu_bench.log 2>&1
python tools/tools_launch_agg.py gpurun_out/r02_c2_launches.csv 4 > gpurun_out/r02_c2_launch_agg.txt
