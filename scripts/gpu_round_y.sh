python -m paper_2509_21527_b200.build > gpurun_out/y_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "rounded" > gpurun_out/y_pytest0.log 2>&1; echo rc=$? >> gpurun_out/y_pytest0.log
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/y_pytest2.log 2>&1; echo rc=$? >> gpurun_out/y_pytest2.log
timeout 600 python bench.py --steps 300 --warmup 20 --zones rounded --no-cpu --no-nccl > gpurun_out/y_bench_C3_n1_rounded.json 2> gpurun_out/y_bench_C3_n1_rounded.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29813 bench.py --gpus 2 --steps 300 --warmup 20 --config C3 --no-cpu > gpurun_out/y_bench_C3_n2.json 2> gpurun_out/y_bench_C3_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29814 bench.py --gpus 2 --steps 300 --warmup 20 --config C3 --no-cpu --zones rounded > gpurun_out/y_bench_C3_n2_rounded.json 2> gpurun_out/y_bench_C3_n2_rounded.err
