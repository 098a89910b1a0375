set -x
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/q_pytest.txt 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/q_pytest.txt
HALO_PROFILE=1 timeout 300 python bench.py > gpurun_out/q_bench1.json 2> gpurun_out/q_bench1.err; echo rc=$?
grep halo_profile gpurun_out/q_bench1.err | tail -2
CMD="python bench.py --steps 20 --warmup 5 --no-cpu --no-graph --no-floors --no-ns --no-fused --no-nccl --no-e2e"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/q_launches.csv $CMD > gpurun_out/q_ncu_l.log 2>&1; echo ncu1_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exchange_ll -s 30 -c 2 -o gpurun_out/q_ncu_full $CMD > gpurun_out/q_ncu_f.log 2>&1; echo ncu2_rc=$?
ls -la gpurun_out/q_ncu_full*
