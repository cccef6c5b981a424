# A/B of the top-k warm start on one GPU (each command bounded by its own timeout)
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x -m gpu > gpurun_out/w_tests.log 2>&1; tail -2 gpurun_out/w_tests.log
for rep in 1 2 3; do
  for v in main nowarm; do
    if [ $v = main ]; then L=paper_1802_08021_b200/libsparcml.so; else L=paper_1802_08021_b200/libvar_$v.so; fi
    echo "== topk $v" >> gpurun_out/w_ab.log
    SPARCML_LIB=$L timeout 60 python tools/topk_phases.py --reps 40 >> gpurun_out/w_ab.log 2>&1
  done
done
SPARCML_LIB=paper_1802_08021_b200/libvar_marks.so timeout 60 python tools/topk_phases.py --reps 40 >> gpurun_out/w_ab.log 2>&1
timeout 600 python bench.py > gpurun_out/w_bench_n1.log 2> gpurun_out/w_bench_n1.err; tail -1 gpurun_out/w_bench_n1.err
