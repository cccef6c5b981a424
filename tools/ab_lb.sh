# A/B: merge look-back polling rounds vs per-thread spin; top-k grid barrier acq_rel vs membar.gl
timeout 500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_allreduce.py tests/test_gpu_f64.py -q -x -m gpu > gpurun_out/l_tests.log 2>&1; tail -2 gpurun_out/l_tests.log
for rep in 1 2 3; do
  for v in main lbspin; do
    if [ $v = main ]; then L=paper_1802_08021_b200/libsparcml.so; else L=paper_1802_08021_b200/libvar_$v.so; fi
    echo "== merge $v" >> gpurun_out/l_ab.log
    SPARCML_LIB=$L timeout 60 python tools/merge_bench.py --reps 30 >> gpurun_out/l_ab.log 2>&1
  done
  for v in main barsc; do
    if [ $v = main ]; then L=paper_1802_08021_b200/libsparcml.so; else L=paper_1802_08021_b200/libvar_$v.so; fi
    echo "== topk $v" >> gpurun_out/l_ab.log
    SPARCML_LIB=$L timeout 60 python tools/topk_phases.py --pre 80 --reps 40 >> gpurun_out/l_ab.log 2>&1
  done
done
SPARCML_LIB=paper_1802_08021_b200/libvar_mmarks.so timeout 60 python tools/merge_bench.py >> gpurun_out/l_ab.log 2>&1
SPARCML_LIB=paper_1802_08021_b200/libvar_marks.so timeout 120 python tools/topk_phases.py --pre 80 --reps 40 >> gpurun_out/l_ab.log 2>&1
