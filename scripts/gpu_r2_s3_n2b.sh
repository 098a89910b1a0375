set -x
python scripts/nvl_probe.py > gpurun_out/n2b_probe.txt 2>&1; cat gpurun_out/n2b_probe.txt | head -40
nvidia-smi nvlink -gt d -i 0 > gpurun_out/n2b_smi.txt 2>&1; head -30 gpurun_out/n2b_smi.txt
nvidia-smi nvlink -h 2>&1 | grep -i "thro\|count\|-gt\|-g " | head -20
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/n2b_pytest.txt 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/n2b_pytest.txt
L=paper_2509_21527_b200/libhalo.so
timeout 1500 python scripts/ab.py --gpus 2 --libs "head=ab/libhalo_head.so,new=$L,hostplan=$L@HALO_PLAN_HOST=1" --config C4-bw8 --reps 2 --steps 200 > gpurun_out/n2b_ab_bw8.txt 2>&1; cut -c1-140 gpurun_out/n2b_ab_bw8.txt
timeout 1500 python scripts/ab.py --gpus 2 --libs "head=ab/libhalo_head.so,new=$L" --config C1 --reps 3 > gpurun_out/n2b_ab_C1.txt 2>&1; cut -c1-140 gpurun_out/n2b_ab_C1.txt
HALO_PROFILE=1 timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu --no-floors --no-graph --no-fused > gpurun_out/n2b_bench1.json 2> gpurun_out/n2b_bench1.err; grep halo_profile gpurun_out/n2b_bench1.err | tail -2
