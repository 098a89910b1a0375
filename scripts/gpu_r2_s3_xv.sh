# x CTA-size variants A/B vs the HEAD build (C3 1 GPU), GPU suite, traces
set -x
L=paper_2509_21527_b200/libhalo.so
timeout 600 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/x_pytest.txt 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/x_pytest.txt
timeout 1200 python scripts/ab.py --libs "head=ab/libhalo_head.so,v1=$L@HALO_X_VARIANT=1,v0=$L@HALO_X_VARIANT=0,v2=$L@HALO_X_VARIANT=2" --config C3 --reps 3 > gpurun_out/x_ab_C3.txt 2>&1; cut -c1-150 gpurun_out/x_ab_C3.txt
for v in 1 2; do HALO_X_VARIANT=$v timeout 120 python scripts/trace.py --config C3 --flush --queue 10 --no-mid-event; done > gpurun_out/x_trace.txt 2>&1; cat gpurun_out/x_trace.txt
timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu --no-floors > gpurun_out/x_bench1.json 2> gpurun_out/x_bench1.err; echo rc=$?
