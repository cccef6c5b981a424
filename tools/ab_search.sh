# A/B: block-wide 129-ary chunk search (main) vs one warp per end, 33-ary (wsearch)
timeout 500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_allreduce.py tests/test_gpu_f64.py tests/test_gpu_fusion.py tests/test_gpu_allgather.py tests/test_gpu_failures.py -q -x -m gpu > gpurun_out/s_tests.log 2>&1; tail -2 gpurun_out/s_tests.log
for rep in 1 2 3; do
  for v in main wsearch; do
    if [ $v = main ]; then L=paper_1802_08021_b200/libsparcml.so; else L=paper_1802_08021_b200/libvar_$v.so; fi
    echo "== merge $v" >> gpurun_out/s_ab.log
    SPARCML_LIB=$L timeout 60 python tools/merge_bench.py --reps 30 >> gpurun_out/s_ab.log 2>&1
  done
done
SPARCML_LIB=paper_1802_08021_b200/libvar_mmarks.so timeout 60 python tools/merge_bench.py >> gpurun_out/s_ab.log 2>&1
timeout 600 python bench.py --config cfg3 > gpurun_out/s_bench_cfg3_n1.log 2>&1
