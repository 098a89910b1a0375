python -m paper_2509_21527_b200.build > gpurun_out/w_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_migrate.py -x -q > gpurun_out/w_pytest0.log 2>&1; echo rc=$? >> gpurun_out/w_pytest0.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > gpurun_out/w_pytest1.log 2>&1; echo rc=$? >> gpurun_out/w_pytest1.log
