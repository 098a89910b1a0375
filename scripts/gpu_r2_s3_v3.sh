set -x
L=paper_2509_21527_b200/libhalo.so
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/v3_pytest.txt 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/v3_pytest.txt
timeout 1800 python scripts/ab.py --libs "head=ab/libhalo_head.so,new=$L,hostplan=$L@HALO_PLAN_HOST=1" --config C3 --reps 4 > gpurun_out/v3_ab_C3.txt 2>&1; cut -c1-140 gpurun_out/v3_ab_C3.txt
HALO_PROFILE=1 timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu --no-floors > gpurun_out/v3_bench1.json 2> gpurun_out/v3_bench1.err; echo rc=$?
grep halo_profile gpurun_out/v3_bench1.err | tail -2
