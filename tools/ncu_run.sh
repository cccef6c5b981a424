# ncu --set full captures (one launch each, source-level) of the top-k and the merge
NCU=/usr/local/cuda/bin/ncu
timeout 300 $NCU --set full --import-source on --clock-control none -k regex:topk_stream -s 5 -c 1 -f -o gpurun_out/r2_topk_src python tools/topk_phases.py --reps 3 > gpurun_out/ncu_topk.log 2>&1
timeout 300 $NCU --set full --import-source on --clock-control none -k regex:merge_jobs -s 3 -c 1 -f -o gpurun_out/r2_merge_src python tools/merge_bench.py --reps 2 > gpurun_out/ncu_merge.log 2>&1
ls -la gpurun_out/*.ncu-rep
