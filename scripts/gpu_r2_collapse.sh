# hop-group (collapsed) LL plan: full GPU suite, per-CTA traces, C3 bench at N=1 and N=2
set -x
export HALO_G3_LOG=gpurun_out/c_g3.jsonl
rm -f $HALO_G3_LOG
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/c_pytest.txt 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/c_pytest.txt
timeout 120 python scripts/trace.py --config C3 --flush --queue 10 > gpurun_out/c_trace.txt 2>&1
timeout 120 python scripts/trace.py --config C3 --flush --queue 10 --fused > gpurun_out/c_trace_fused.txt 2>&1
HALO_COLLAPSE=0 timeout 120 python scripts/trace.py --config C3 --flush --queue 10 > gpurun_out/c_trace_staged.txt 2>&1
timeout 300 python bench.py --steps 300 --no-ns --no-cpu --no-floors > gpurun_out/c_bench1.json 2> gpurun_out/c_bench1.err; echo bench1_rc=$?
tail -3 gpurun_out/c_bench1.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 300 --no-ns --no-floors > gpurun_out/c_bench2.json 2> gpurun_out/c_bench2.err; echo bench2_rc=$?
tail -3 gpurun_out/c_bench2.err
