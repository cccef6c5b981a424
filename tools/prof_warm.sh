# steady-state (warm-start) top-k: phase marks and one ncu --set full capture; merge marks
NCU=/usr/local/cuda/bin/ncu
SPARCML_LIB=paper_1802_08021_b200/libvar_marks.so timeout 120 python tools/topk_phases.py --pre 80 --reps 40 > gpurun_out/p_phases.log 2>&1
timeout 120 python tools/topk_phases.py --pre 80 --reps 40 >> gpurun_out/p_phases.log 2>&1
timeout 300 $NCU --set full --import-source on --clock-control none -k regex:topk_stream -s 80 -c 1 -f -o gpurun_out/p_topk python tools/topk_phases.py --pre 80 --reps 3 > gpurun_out/p_ncu_topk.log 2>&1
timeout 300 $NCU --set full --import-source on --clock-control none -k regex:merge_jobs -s 3 -c 1 -f -o gpurun_out/p_merge python tools/merge_bench.py --reps 2 > gpurun_out/p_ncu_merge.log 2>&1
ls -la gpurun_out
