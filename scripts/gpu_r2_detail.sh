set -x
HALO_DEBUG=8192 timeout 120 python scripts/trace.py --config C3 --flush --queue 10 > gpurun_out/d_trace.txt 2>&1
HALO_DEBUG=8192 timeout 120 python scripts/trace.py --config C3 --flush --queue 10 --no-fshift > gpurun_out/d_trace_nofs.txt 2>&1
timeout 120 python scripts/trace.py --config C3 --flush --queue 10 > gpurun_out/d_trace_plain.txt 2>&1
tail -2 gpurun_out/d_trace.txt
