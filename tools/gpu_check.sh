python bench.py --config c1b --steps 10 --warmup 3 > gpurun_out/r02_bench_c1b.json 2> gpurun_out/r02_bench_c1b.err
python bench.py --config c1b --precision f64 --steps 10 --warmup 3 > gpurun_out/r02_bench_c1b_f64.json 2> gpurun_out/r02_bench_c1b_f64.err
