set -x
python -m paper_2509_21527_b200.build > gpurun_out/ce_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ce" > gpurun_out/ce_pytest1.log 2>&1; echo rc=$? >> gpurun_out/ce_pytest1.log
timeout 600 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/ce_pytest2.log 2>&1; echo rc=$? >> gpurun_out/ce_pytest2.log
for cfg in C1 C4-1D C4-bw2 C4-bw5 C4-bw8; do for proto in ll ce; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 300 --warmup 20 --config $cfg --proto $proto --no-graph > gpurun_out/ce_bench_${cfg}_${proto}.json 2> gpurun_out/ce_bench_${cfg}_${proto}.err
done; done
