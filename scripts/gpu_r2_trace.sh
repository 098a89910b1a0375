# per-CTA trace of one C3 step on 1 GPU: collapsed plan, fused, without fshift, and staged
set -x
python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x -k "mutation or timers" > gpurun_out/t_pytest.txt 2>&1; echo rc=$?; tail -3 gpurun_out/t_pytest.txt
timeout 120 python scripts/trace.py --config C3 --flush --queue 10 > gpurun_out/t_trace.txt 2>&1
timeout 120 python scripts/trace.py --config C3 --flush --queue 10 --no-fshift > gpurun_out/t_trace_nofs.txt 2>&1
timeout 120 python scripts/trace.py --config C3 --flush --queue 10 --fused > gpurun_out/t_trace_fused.txt 2>&1
HALO_COLLAPSE=0 timeout 120 python scripts/trace.py --config C3 --flush --queue 10 > gpurun_out/t_trace_staged.txt 2>&1
tail -c 3000 gpurun_out/t_trace.txt
