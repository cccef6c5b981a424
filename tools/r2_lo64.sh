timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -m gpu > gpurun_out/k_tests.log 2>&1; tail -2 gpurun_out/k_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/k_smoke.log 2>&1; tail -1 gpurun_out/k_smoke.log
timeout 600 python bench.py > gpurun_out/k_bench_n1.log 2> gpurun_out/k_bench_n1.err
