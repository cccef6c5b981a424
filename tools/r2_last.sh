# last re-check of the final build on a 2-GPU box
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/h_tests.log 2>&1; tail -2 gpurun_out/h_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1; tail -1 gpurun_out/h_smoke.log
timeout 600 python bench.py > gpurun_out/h_bench_n1.log 2> gpurun_out/h_bench_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 > gpurun_out/h_bench_n2.log 2> gpurun_out/h_bench_n2.err
timeout 120 python tools/merge_bench.py --reps 30 > gpurun_out/h_merge.log 2>&1
SPARCML_LIB=paper_1802_08021_b200/libvar_mmarks.so timeout 60 python tools/merge_bench.py >> gpurun_out/h_merge.log 2>&1
timeout 300 $NCU --set full --import-source on --clock-control none -k regex:merge_jobs -s 3 -c 1 -f -o gpurun_out/h_merge python tools/merge_bench.py --reps 2 > gpurun_out/h_ncu_merge.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/h_launches.csv python bench.py --steps 5 --warmup 3 > gpurun_out/h_ncu_list.log 2>&1
