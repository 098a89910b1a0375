# build, parity (1 and 2 GPUs), benches incl. the bandwidth probes
python -m paper_2509_21527_b200.build > gpurun_out/b_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/b_pytest1.log 2>&1; echo rc=$? >> gpurun_out/b_pytest1.log
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/b_pytest2.log 2>&1; echo rc=$? >> gpurun_out/b_pytest2.log
timeout 300 python bench.py --steps 300 --warmup 20 --no-graph --no-cpu > gpurun_out/b_bench_C3_n1.json 2> gpurun_out/b_bench_C3_n1.err
for run in "C1 ll" "C4-1D ll" "C4-1D ce" "C4-bw8 ll" "C4-bw8 ce" "C4-bw8 paper" "C4-bw2 ll"; do
set -- $run
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 300 --warmup 20 --config $1 --proto $2 --no-graph > gpurun_out/b_bench_$1_$2.json 2> gpurun_out/b_bench_$1_$2.err
done
