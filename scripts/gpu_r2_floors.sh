# round-2 check: new GPU tests, default bench N=1, N=2 floors (t(B), bandwidth), C1 NCCL eager+graph
set -x
timeout 600 python -m pytest tests/test_gpu_assign.py tests/test_abi.py -x -q -m gpu -p no:cacheprovider > gpurun_out/f_pytest.txt 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/f_pytest.txt
timeout 400 python bench.py > gpurun_out/f_bench1.json 2> gpurun_out/f_bench1.err; echo bench1_rc=$?
tail -5 gpurun_out/f_bench1.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --no-ns > gpurun_out/f_bench2.json 2> gpurun_out/f_bench2.err; echo bench2_rc=$?
tail -5 gpurun_out/f_bench2.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config C1 --no-ns --no-floors > gpurun_out/f_bench2_c1.json 2> gpurun_out/f_bench2_c1.err; echo bench2c1_rc=$?
tail -5 gpurun_out/f_bench2_c1.err
ncu --query-metrics 2>/dev/null | grep -i "nvl" > gpurun_out/f_ncu_nvl_metrics.txt; wc -l gpurun_out/f_ncu_nvl_metrics.txt
nvidia-smi nvlink -s -i 0 > gpurun_out/f_nvlink_status.txt 2>&1; head -5 gpurun_out/f_nvlink_status.txt
