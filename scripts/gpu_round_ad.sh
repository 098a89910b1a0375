python -m paper_2509_21527_b200.build > gpurun_out/ad_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_migrate.py -x -q > gpurun_out/ad_pytest1.log 2>&1; echo rc=$? >> gpurun_out/ad_pytest1.log
