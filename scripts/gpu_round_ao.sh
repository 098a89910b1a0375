# the 8-process path (one DD rank per process) on a 4-GPU box: 2 processes per GPU, gloo for the
# host collectives (NCCL refuses two ranks on one GPU); a functional check, not a bench value
python -m paper_2509_21527_b200.build > gpurun_out/ao_build.log 2>&1
for c in C3 C5 C4-3D; do
HALO_BENCH_PG=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port $((29900 + RANDOM % 90)) bench.py --gpus 8 --steps 200 --warmup 10 --config $c --no-nccl --no-cpu > gpurun_out/ao_bench_${c}_n8.json 2> gpurun_out/ao_bench_${c}_n8.err
done
