python -m paper_2509_21527_b200.build > gpurun_out/ab_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_pme.py -x -q > gpurun_out/ab_pytest0.log 2>&1; echo rc=$? >> gpurun_out/ab_pytest0.log
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -k "pme or migrate" > gpurun_out/ab_pytest2.log 2>&1; echo rc=$? >> gpurun_out/ab_pytest2.log
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu --no-graph --no-nccl --pme > gpurun_out/ab_bench_C3_n1.json 2> gpurun_out/ab_bench_C3_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29851 bench.py --gpus 2 --steps 200 --warmup 10 --config C3 --no-cpu --no-graph --no-nccl --pme > gpurun_out/ab_bench_C3_n2.json 2> gpurun_out/ab_bench_C3_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29852 bench.py --gpus 2 --steps 200 --warmup 10 --config C4-1D --no-cpu --no-graph --no-nccl --pme > gpurun_out/ab_bench_C41D_n2.json 2> gpurun_out/ab_bench_C41D_n2.err
