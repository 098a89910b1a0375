python -m paper_2509_21527_b200.build > gpurun_out/z_build.log 2>&1
HALO_PROFILE=1 timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu --no-graph > gpurun_out/z_bench_C3_n1.json 2> gpurun_out/z_bench_C3_n1.err
HALO_PROFILE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29815 bench.py --gpus 2 --steps 100 --warmup 10 --config C4-1D --no-cpu --no-graph --no-nccl > gpurun_out/z_bench_C41D_n2.json 2> gpurun_out/z_bench_C41D_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29816 bench.py --gpus 2 --steps 100 --warmup 10 --config C1 --no-cpu --no-graph --no-nccl > gpurun_out/z_bench_C1_n2.json 2> gpurun_out/z_bench_C1_n2.err
