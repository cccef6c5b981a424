# full check on a 2-GPU box: GPU suite (incl. the IPC world), smoke, bench N=1 and N=2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c_tests.log 2>&1; tail -3 gpurun_out/c_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c_smoke.log 2>&1; tail -1 gpurun_out/c_smoke.log
timeout 600 python bench.py > gpurun_out/c_bench_n1.log 2> gpurun_out/c_bench_n1.err; tail -1 gpurun_out/c_bench_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 > gpurun_out/c_bench_n2.log 2> gpurun_out/c_bench_n2.err; tail -1 gpurun_out/c_bench_n2.err
SPARCML_LIB=paper_1802_08021_b200/libvar_marks.so timeout 60 python tools/topk_phases.py > gpurun_out/c_phases.log 2>&1
timeout 60 python tools/topk_phases.py --reps 40 >> gpurun_out/c_phases.log 2>&1
