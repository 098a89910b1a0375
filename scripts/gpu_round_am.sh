python -m paper_2509_21527_b200.build > gpurun_out/am_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_migrate.py tests/test_gpu_pme.py -q > gpurun_out/am_pytest.log 2>&1; echo rc=$? >> gpurun_out/am_pytest.log
