# A/B: packed-word look-back (main) vs the flag + acquire version (lbspin)
timeout 500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_allreduce.py tests/test_gpu_f64.py tests/test_gpu_fusion.py -q -x -m gpu > gpurun_out/l2_tests.log 2>&1; tail -2 gpurun_out/l2_tests.log
SPARCML_LIB=paper_1802_08021_b200/libvar_mchecks.so timeout 500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_allreduce.py -q -x -m gpu -k "merge or rd or RD or recursive" > gpurun_out/l2_tests_checks.log 2>&1; tail -2 gpurun_out/l2_tests_checks.log
for rep in 1 2 3; do
  for v in main lbspin; do
    if [ $v = main ]; then L=paper_1802_08021_b200/libsparcml.so; else L=paper_1802_08021_b200/libvar_$v.so; fi
    echo "== merge $v" >> gpurun_out/l2_ab.log
    SPARCML_LIB=$L timeout 60 python tools/merge_bench.py --reps 30 >> gpurun_out/l2_ab.log 2>&1
  done
done
SPARCML_LIB=paper_1802_08021_b200/libvar_mmarks.so timeout 60 python tools/merge_bench.py >> gpurun_out/l2_ab.log 2>&1
timeout 600 python bench.py --config cfg3 > gpurun_out/l2_bench_cfg3.log 2>&1
