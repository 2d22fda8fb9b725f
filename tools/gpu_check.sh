timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02_bench_c2_reference.json 2> gpurun_out/r02_ref.err
