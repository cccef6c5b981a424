# round-2 final re-check on a 4-GPU box: GPU suite (IPC world at 4), smoke, bench cfg2 at N=1/2/4 and
# the reference arm, the other workloads at N=1, merge and top-k diagnostics, ncu launch list + captures
NCU=/usr/local/cuda/bin/ncu
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g_tests.log 2>&1; tail -2 gpurun_out/g_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; tail -1 gpurun_out/g_smoke.log
timeout 600 python bench.py > gpurun_out/g_bench_n1.log 2> gpurun_out/g_bench_n1.err
timeout 600 $TR --nproc-per-node 2 --master-port 29512 bench.py --gpus 2 > gpurun_out/g_bench_n2.log 2> gpurun_out/g_bench_n2.err
timeout 600 $TR --nproc-per-node 4 --master-port 29513 bench.py --gpus 4 > gpurun_out/g_bench_n4.log 2> gpurun_out/g_bench_n4.err
timeout 600 python bench.py --impl reference > gpurun_out/g_bench_ref_n1.log 2>&1
for c in cfg1 cfg3 cfg4 cfg5 bucket512; do timeout 600 python bench.py --config $c > gpurun_out/g_bench_${c}_n1.log 2>&1; done
timeout 600 $TR --nproc-per-node 4 --master-port 29514 bench.py --gpus 4 --config cfg4 > gpurun_out/g_bench_cfg4_n4.log 2>&1
timeout 600 $TR --nproc-per-node 4 --master-port 29515 bench.py --gpus 4 --config cfg3 > gpurun_out/g_bench_cfg3_n4.log 2>&1
timeout 120 python tools/merge_bench.py --reps 30 > gpurun_out/g_merge.log 2>&1
SPARCML_LIB=paper_1802_08021_b200/libvar_mmarks.so timeout 60 python tools/merge_bench.py >> gpurun_out/g_merge.log 2>&1
timeout 120 python tools/topk_phases.py --pre 80 --reps 40 > gpurun_out/g_phases.log 2>&1
SPARCML_LIB=paper_1802_08021_b200/libvar_marks.so timeout 120 python tools/topk_phases.py --pre 80 --reps 40 >> gpurun_out/g_phases.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g_launches.csv python bench.py --steps 5 --warmup 3 > gpurun_out/g_ncu_list.log 2>&1
timeout 300 $NCU --set full --import-source on --clock-control none -k regex:topk_stream -s 80 -c 1 -f -o gpurun_out/g_topk python tools/topk_phases.py --pre 80 --reps 3 > gpurun_out/g_ncu_topk.log 2>&1
timeout 300 $NCU --set full --import-source on --clock-control none -k regex:merge_jobs -s 3 -c 1 -f -o gpurun_out/g_merge python tools/merge_bench.py --reps 2 > gpurun_out/g_ncu_merge.log 2>&1
ls gpurun_out
