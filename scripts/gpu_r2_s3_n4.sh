# 4 GPUs: multi-process tests + bench lines (C3, C2 with NCCL, C4-2D, C5)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -m gpu -p no:cacheprovider > gpurun_out/n4_pytest.txt 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/n4_pytest.txt
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29611 bench.py --gpus 4 > gpurun_out/n4_bench_C3.json 2> gpurun_out/n4_bench_C3.err; echo rc=$?
timeout 600 $R --master-port 29612 bench.py --gpus 4 --config C2 --no-ns > gpurun_out/n4_bench_C2.json 2> gpurun_out/n4_bench_C2.err; echo rc=$?
timeout 600 $R --master-port 29613 bench.py --gpus 4 --config C4-2D --no-floors > gpurun_out/n4_bench_C42D.json 2> gpurun_out/n4_bench_C42D.err; echo rc=$?
timeout 600 $R --master-port 29614 bench.py --gpus 4 --config C5 --no-floors --no-ns > gpurun_out/n4_bench_C5.json 2> gpurun_out/n4_bench_C5.err; echo rc=$?
for f in gpurun_out/n4_bench_*.json; do echo $f; tail -c 400 $f; echo; done
