set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x -k "int_forces or fused_xf or real_forces" > gpurun_out/d_pytest.txt 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/d_pytest.txt
HALO_DEBUG=8192 timeout 120 python scripts/trace.py --config C3 --flush --queue 10 > gpurun_out/d_trace.txt 2>&1
timeout 120 python scripts/trace.py --config C3 --flush --queue 10 --fused > gpurun_out/d_trace_fused.txt 2>&1
timeout 300 python bench.py --steps 500 --no-ns --no-cpu --no-floors > gpurun_out/d_bench.json 2> gpurun_out/d_bench.err
