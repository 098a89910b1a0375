# 2 GPUs: multi-process tests, bench C3/C1/C4-1D/C4-bw8 (NVLink counters via NVML), NCCL baseline
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -m gpu -p no:cacheprovider > gpurun_out/n2_pytest.txt 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/n2_pytest.txt
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29511 bench.py --gpus 2 > gpurun_out/n2_bench_C3.json 2> gpurun_out/n2_bench_C3.err; echo rc=$?
timeout 600 $R --master-port 29512 bench.py --gpus 2 --config C1 --no-ns --no-floors > gpurun_out/n2_bench_C1.json 2> gpurun_out/n2_bench_C1.err; echo rc=$?
timeout 600 $R --master-port 29513 bench.py --gpus 2 --config C4-1D --no-floors > gpurun_out/n2_bench_C41D.json 2> gpurun_out/n2_bench_C41D.err; echo rc=$?
timeout 600 $R --master-port 29514 bench.py --gpus 2 --config C4-bw8 --no-ns --no-floors > gpurun_out/n2_bench_bw8.json 2> gpurun_out/n2_bench_bw8.err; echo rc=$?
timeout 600 $R --master-port 29515 bench.py --gpus 2 --config C4-bw8 --no-ns --no-floors --proto ce > gpurun_out/n2_bench_bw8_ce.json 2> gpurun_out/n2_bench_bw8_ce.err; echo rc=$?
for f in gpurun_out/n2_bench_*.json; do echo $f; tail -c 600 $f; done
tail -3 gpurun_out/n2_bench_C3.err
