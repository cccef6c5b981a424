# A/B diagnostics on one GPU (each command bounded by its own timeout)
T="timeout 300"
$T python -m pytest tests/test_gpu_kernels.py -q -x -m gpu > gpurun_out/ab3_tests.log 2>&1; tail -2 gpurun_out/ab3_tests.log
for rep in 1 2; do
  for v in main oldfind; do
    if [ $v = main ]; then L=paper_1802_08021_b200/libsparcml.so; else L=paper_1802_08021_b200/libvar_$v.so; fi
    echo "== topk $v" >> gpurun_out/ab3.log
    SPARCML_LIB=$L timeout 60 python tools/topk_phases.py --reps 30 >> gpurun_out/ab3.log 2>&1
  done
done
echo "== merge main" >> gpurun_out/ab3.log
timeout 60 python tools/merge_bench.py >> gpurun_out/ab3.log 2>&1
SPARCML_LIB=paper_1802_08021_b200/libvar_marks.so timeout 60 python tools/topk_phases.py >> gpurun_out/ab3.log 2>&1
$T python -m pytest tests/test_gpu_allreduce.py tests/test_gpu_f64.py tests/test_gpu_fusion.py -q -x -m gpu > gpurun_out/ab3_tests_ar.log 2>&1; tail -2 gpurun_out/ab3_tests_ar.log
