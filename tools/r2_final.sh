# round-2 re-check on a 2-GPU box: GPU suite (incl. the IPC world), smoke, bench N=1/N=2,
# top-k phases, ncu launch list of the bench and one --set full capture of the top-k
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f_tests.log 2>&1; tail -2 gpurun_out/f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; tail -1 gpurun_out/f_smoke.log
timeout 600 python bench.py > gpurun_out/f_bench_n1.log 2> gpurun_out/f_bench_n1.err; tail -1 gpurun_out/f_bench_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 > gpurun_out/f_bench_n2.log 2> gpurun_out/f_bench_n2.err; tail -1 gpurun_out/f_bench_n2.err
timeout 600 python bench.py --impl reference > gpurun_out/f_bench_ref_n1.log 2> gpurun_out/f_bench_ref_n1.err; tail -1 gpurun_out/f_bench_ref_n1.err
timeout 60 python tools/topk_phases.py --reps 40 > gpurun_out/f_phases.log 2>&1
SPARCML_LIB=paper_1802_08021_b200/libvar_marks.so timeout 60 python tools/topk_phases.py --reps 40 >> gpurun_out/f_phases.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 5 --warmup 3 > gpurun_out/f_ncu_list.log 2>&1
timeout 300 $NCU --set full --import-source on --clock-control none -k regex:topk_stream -s 5 -c 1 -f -o gpurun_out/f_topk python tools/topk_phases.py --reps 3 > gpurun_out/f_ncu_topk.log 2>&1
ls -la gpurun_out/
