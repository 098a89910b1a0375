python -m paper_2509_21527_b200.build > gpurun_out/af_build.log 2>&1
timeout 300 python scripts/trace.py --config C3 --flush --queue 10 > gpurun_out/af_trace_C3_n1.txt 2>&1
timeout 300 python scripts/trace.py --config C3 --flush --queue 10 --no-fshift > gpurun_out/af_trace_C3_n1_nofs.txt 2>&1
timeout 300 python scripts/trace.py --config C5 --flush --queue 10 > gpurun_out/af_trace_C5_n1.txt 2>&1
