timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/z_tests.log 2>&1; tail -2 gpurun_out/z_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.log 2>&1; tail -1 gpurun_out/z_smoke.log
timeout 600 python bench.py > gpurun_out/z_bench_n1.log 2> gpurun_out/z_bench_n1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/z_bench_ref.log 2>&1
