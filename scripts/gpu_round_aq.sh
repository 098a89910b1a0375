python -m paper_2509_21527_b200.build > gpurun_out/aq_build.log 2>&1
timeout 300 python scripts/trace.py --config C3 --flush --queue 10 --no-mid-event > gpurun_out/aq_trace_C3_n1.txt 2>&1
timeout 300 python scripts/trace.py --config C3 --flush --queue 10 --no-mid-event --no-fshift > gpurun_out/aq_trace_C3_n1_nofs.txt 2>&1
timeout 300 python scripts/trace.py --config C3 --flush --queue 10 > gpurun_out/aq_trace_C3_n1_mid.txt 2>&1
