timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err
python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err
python tools/tools_sol.py c2 bf16 > gpurun_out/r02_c2_sol_bf16.txt 2>&1
python tools/tools_shape_profile.py c2 bf16 > gpurun_out/r02_c2_shape_profile.txt 2>&1
