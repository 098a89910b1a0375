set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
export HALO_G3_LOG=gpurun_out/v_g3.jsonl
rm -f $HALO_G3_LOG
timeout 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/v_pytest.txt 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/v_pytest.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.txt 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/v_smoke.txt
timeout 300 python bench.py > gpurun_out/v_bench1.json 2> gpurun_out/v_bench1.err; echo bench1_rc=$?
tail -c 1500 gpurun_out/v_bench1.json; tail -5 gpurun_out/v_bench1.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/v_bench2.json 2> gpurun_out/v_bench2.err; echo bench2_rc=$?
tail -c 1500 gpurun_out/v_bench2.json; tail -5 gpurun_out/v_bench2.err
