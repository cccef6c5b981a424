# top-k warm-miss tests, the merge's cp.async staging A/B, bench N=1 (one GPU, each step bounded)
timeout 400 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_allreduce.py -q -x -m gpu > gpurun_out/m_tests.log 2>&1; tail -2 gpurun_out/m_tests.log
for rep in 1 2 3; do
  for v in main msync; do
    if [ $v = main ]; then L=paper_1802_08021_b200/libsparcml.so; else L=paper_1802_08021_b200/libvar_$v.so; fi
    echo "== merge $v" >> gpurun_out/m_ab.log
    SPARCML_LIB=$L timeout 60 python tools/merge_bench.py --reps 30 >> gpurun_out/m_ab.log 2>&1
  done
done
SPARCML_LIB=paper_1802_08021_b200/libvar_mmarks.so timeout 60 python tools/merge_bench.py >> gpurun_out/m_ab.log 2>&1
timeout 600 python bench.py > gpurun_out/m_bench_n1.log 2> gpurun_out/m_bench_n1.err; tail -1 gpurun_out/m_bench_n1.err
timeout 600 python bench.py --config cfg3 > gpurun_out/m_bench_cfg3.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/m_launches.csv python bench.py --steps 5 --warmup 3 > gpurun_out/m_ncu_list.log 2>&1
