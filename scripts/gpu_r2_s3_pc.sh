set -x
HALO_PLAN_CHECK=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "int_forces and ll and not staged and (T3D or C1 or W2)" > gpurun_out/pc_pytest.txt 2>&1; echo rc=$?
grep -a "plan_check" gpurun_out/pc_pytest.txt | head -40; tail -5 gpurun_out/pc_pytest.txt
HALO_PLAN_CHECK=1 timeout 300 python -m pytest tests/test_gpu_fuzz.py -x -q -m gpu -p no:cacheprovider -k "test_fuzz_parity and ll" > gpurun_out/pc_fuzz.txt 2>&1; echo rc=$?
grep -a "plan_check" gpurun_out/pc_fuzz.txt | head -40; tail -5 gpurun_out/pc_fuzz.txt
