python -m paper_2509_21527_b200.build > gpurun_out/aa_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_migrate.py -x -q > gpurun_out/aa_pytest1.log 2>&1; echo rc=$? >> gpurun_out/aa_pytest1.log
HALO_PROFILE=1 timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu --no-graph > gpurun_out/aa_bench_C3_n1.json 2> gpurun_out/aa_bench_C3_n1.err
for pr in auto ll ce; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29820 + RANDOM % 100)) bench.py --gpus 2 --steps 200 --warmup 10 --config C4-bw8 --no-cpu --no-graph --no-nccl --no-ns --proto $pr > gpurun_out/aa_bench_C4bw8_$pr.json 2> gpurun_out/aa_bench_C4bw8_$pr.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29820 + RANDOM % 100)) bench.py --gpus 2 --steps 200 --warmup 10 --config C4-bw5 --no-cpu --no-graph --no-nccl --no-ns --proto $pr > gpurun_out/aa_bench_C4bw5_$pr.json 2> gpurun_out/aa_bench_C4bw5_$pr.err
done
