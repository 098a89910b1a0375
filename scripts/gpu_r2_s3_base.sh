# round 2 (session 3): full GPU suite on 2 GPUs (multi-process tests run), smoke, bench N=1/N=2, launch list N=1
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/s3_pytest.txt 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/s3_pytest.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.txt 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/s3_smoke.txt
timeout 400 python bench.py > gpurun_out/s3_bench1.json 2> gpurun_out/s3_bench1.err; echo bench1_rc=$?
tail -5 gpurun_out/s3_bench1.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/s3_bench2.json 2> gpurun_out/s3_bench2.err; echo bench2_rc=$?
tail -5 gpurun_out/s3_bench2.err
CMD="python bench.py --steps 20 --warmup 5 --no-cpu --no-graph --no-floors --no-ns --no-fused --no-nccl"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s3_launches.csv $CMD > gpurun_out/s3_ncu_l.log 2>&1; echo ncu_rc=$?
