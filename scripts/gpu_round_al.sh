python -m paper_2509_21527_b200.build > gpurun_out/al_build.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/al_pytest.log 2>&1; echo rc=$? >> gpurun_out/al_pytest.log
