set -x
L=paper_2509_21527_b200/libhalo.so
timeout 600 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/y_pytest.txt 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/y_pytest.txt
timeout 1200 python scripts/ab.py --libs "head=ab/libhalo_head.so,new=$L" --config C3 --reps 4 > gpurun_out/y_ab_C3.txt 2>&1; cut -c1-150 gpurun_out/y_ab_C3.txt
HALO_DEBUG=8192 timeout 120 python scripts/trace.py --config C3 --flush --queue 10 --no-mid-event > gpurun_out/y_trace.txt 2>&1; cat gpurun_out/y_trace.txt
HALO_PROFILE=1 timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu --no-floors > gpurun_out/y_bench1.json 2> gpurun_out/y_bench1.err; echo rc=$?
grep halo_profile gpurun_out/y_bench1.err | tail -3
