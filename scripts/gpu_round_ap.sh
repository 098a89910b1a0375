python -m paper_2509_21527_b200.build > gpurun_out/ap_build.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_multiproc.py -q > gpurun_out/ap_pytest_mp.log 2>&1; echo rc=$? >> gpurun_out/ap_pytest_mp.log
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu > gpurun_out/ap_bench_n1.json 2> gpurun_out/ap_bench_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29881 bench.py --gpus 4 --steps 200 --warmup 10 > gpurun_out/ap_bench_n4.json 2> gpurun_out/ap_bench_n4.err
