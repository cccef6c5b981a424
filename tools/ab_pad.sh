# A/B: padded merge windows (main) vs unpadded (nopad); 32-byte status entries
timeout 500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_allreduce.py tests/test_gpu_f64.py tests/test_gpu_fusion.py tests/test_gpu_allgather.py -q -x -m gpu > gpurun_out/pd_tests.log 2>&1; tail -2 gpurun_out/pd_tests.log
for rep in 1 2 3; do
  for v in main nopad lbspin; do
    if [ $v = main ]; then L=paper_1802_08021_b200/libsparcml.so; else L=paper_1802_08021_b200/libvar_$v.so; fi
    echo "== merge $v" >> gpurun_out/pd_ab.log
    SPARCML_LIB=$L timeout 60 python tools/merge_bench.py --reps 30 >> gpurun_out/pd_ab.log 2>&1
  done
done
SPARCML_LIB=paper_1802_08021_b200/libvar_mmarks.so timeout 60 python tools/merge_bench.py >> gpurun_out/pd_ab.log 2>&1
timeout 300 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:merge_jobs -s 3 -c 1 -f -o gpurun_out/pd_merge python tools/merge_bench.py --reps 2 > gpurun_out/pd_ncu_merge.log 2>&1
