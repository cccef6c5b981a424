timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_algorithm1.py tests/test_gpu_lr.py -q -x -m gpu > gpurun_out/j_tests.log 2>&1; tail -2 gpurun_out/j_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j_smoke.log 2>&1; tail -1 gpurun_out/j_smoke.log
timeout 600 python bench.py > gpurun_out/j_bench_n1.log 2> gpurun_out/j_bench_n1.err
timeout 600 python bench.py --config cfg3 > gpurun_out/j_bench_cfg3_n1.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/j_launches.csv python bench.py --steps 5 --warmup 3 > gpurun_out/j_ncu_list.log 2>&1
