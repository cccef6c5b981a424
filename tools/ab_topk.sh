set -x
python -m pytest tests/test_gpu_kernels.py -q -x -m gpu > gpurun_out/ab_tests.log 2>&1
tail -2 gpurun_out/ab_tests.log
for rep in 1 2; do
for v in main r0b0 r1b0 r0b1 nocoop; do
  if [ $v = main ]; then L=paper_1802_08021_b200/libsparcml.so; else L=paper_1802_08021_b200/libvar_$v.so; fi
  echo "== $v" >> gpurun_out/ab_topk.log
  SPARCML_LIB=$L python tools/topk_phases.py --reps 30 >> gpurun_out/ab_topk.log 2>&1
done
done
SPARCML_LIB=paper_1802_08021_b200/libvar_marks.so python tools/topk_phases.py >> gpurun_out/ab_topk.log 2>&1
SPARCML_LIB=paper_1802_08021_b200/libvar_nocoop.so python -m pytest tests/test_gpu_kernels.py -q -x -m gpu -k topk > gpurun_out/ab_tests_nocoop.log 2>&1
tail -2 gpurun_out/ab_tests_nocoop.log
