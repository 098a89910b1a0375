python -m paper_2509_21527_b200.build > gpurun_out/x_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/x_pytest2.log 2>&1; echo rc=$? >> gpurun_out/x_pytest2.log
timeout 600 python bench.py --steps 300 --warmup 20 > gpurun_out/x_bench_C3_n1.json 2> gpurun_out/x_bench_C3_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29811 bench.py --gpus 2 --steps 300 --warmup 20 --config C1 > gpurun_out/x_bench_C1_n2.json 2> gpurun_out/x_bench_C1_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29812 bench.py --gpus 2 --steps 300 --warmup 20 --config C4-1D --no-cpu > gpurun_out/x_bench_C41D_n2.json 2> gpurun_out/x_bench_C41D_n2.err
