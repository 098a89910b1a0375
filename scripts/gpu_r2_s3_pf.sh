# prefetch A/B (C3 1 GPU), GPU suite, e2e packed, set_maps profile, traces
set -x
L=paper_2509_21527_b200/libhalo.so
timeout 600 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/p_pytest.txt 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/p_pytest.txt
timeout 900 python scripts/ab.py --libs "pf=$L,nopf=$L@HALO_PREFETCH=0" --config C3 --reps 4 > gpurun_out/p_ab_C3.txt 2>&1; cat gpurun_out/p_ab_C3.txt | grep -v runs\" ; grep '"lib"' gpurun_out/p_ab_C3.txt | cut -c1-200
HALO_PROFILE=1 timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu --no-floors > gpurun_out/p_bench1.json 2> gpurun_out/p_bench1.err; echo rc=$?
grep halo_profile gpurun_out/p_bench1.err | tail -4
timeout 120 python scripts/trace.py --config C3 --flush --queue 10 --no-mid-event > gpurun_out/p_trace.txt 2>&1; cat gpurun_out/p_trace.txt
HALO_PREFETCH=0 timeout 120 python scripts/trace.py --config C3 --flush --queue 10 --no-mid-event > gpurun_out/p_trace_nopf.txt 2>&1; cat gpurun_out/p_trace_nopf.txt
