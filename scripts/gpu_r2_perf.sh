# C3 on 1 GPU: parity subset, trace (two launches / fused), bench default and with the persisting-L2 plan
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x -k "int_forces or fused or graph or real_forces" > gpurun_out/p_pytest.txt 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/p_pytest.txt
timeout 120 python scripts/trace.py --config C3 --flush --queue 10 > gpurun_out/p_trace.txt 2>&1
timeout 120 python scripts/trace.py --config C3 --flush --queue 10 --fused > gpurun_out/p_trace_fused.txt 2>&1
for i in 1 2; do
timeout 300 python bench.py --steps 500 --no-ns --no-cpu --no-floors > gpurun_out/p_bench_$i.json 2> gpurun_out/p_bench_$i.err
timeout 300 python bench.py --steps 500 --no-ns --no-cpu --no-floors --l2-persist > gpurun_out/p_bench_l2_$i.json 2> gpurun_out/p_bench_l2_$i.err
done
