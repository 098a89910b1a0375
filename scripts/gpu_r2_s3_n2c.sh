set -x
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29811 bench.py --gpus 2 --config C4-2D --no-floors --no-ns --no-e2e --no-nccl > gpurun_out/n2c_C42D.json 2> gpurun_out/n2c_C42D.err; echo rc=$?
tail -c 400 gpurun_out/n2c_C42D.json; grep -a "Error" gpurun_out/n2c_C42D.err | tail -3
timeout 600 $R --master-port 29812 bench.py --gpus 2 --config C4-3D --no-floors --no-ns --no-e2e --no-nccl > gpurun_out/n2c_C43D.json 2> gpurun_out/n2c_C43D.err; echo rc=$?
tail -c 400 gpurun_out/n2c_C43D.json; grep -a "Error" gpurun_out/n2c_C43D.err | tail -3
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/n2c_pytest.txt 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/n2c_pytest.txt
