# final build on 4 GPUs: GPU suite (IPC world at 4), bench cfg2 and cfg3 at N=4
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/i_tests.log 2>&1; tail -2 gpurun_out/i_tests.log
timeout 600 $TR --nproc-per-node 4 --master-port 29513 bench.py --gpus 4 > gpurun_out/i_bench_n4.log 2> gpurun_out/i_bench_n4.err
timeout 600 $TR --nproc-per-node 4 --master-port 29515 bench.py --gpus 4 --config cfg3 > gpurun_out/i_bench_cfg3_n4.log 2>&1
timeout 600 $TR --nproc-per-node 4 --master-port 29516 bench.py --gpus 4 --config cfg4 > gpurun_out/i_bench_cfg4_n4.log 2>&1
