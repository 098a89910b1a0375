set -x
L=paper_2509_21527_b200/libhalo.so
timeout 1200 python scripts/ab.py --libs "xf4=$L,xf3=ab/libhalo_xf3.so" --config C3 --reps 2 > gpurun_out/xf3_ab.txt 2>&1; cut -c1-170 gpurun_out/xf3_ab.txt
HALO_LIB_PATH=ab/libhalo_xf3.so timeout 120 python scripts/trace.py --config C3 --flush --queue 10 --fused > gpurun_out/xf3_trace.txt 2>&1; grep '^{' gpurun_out/xf3_trace.txt | cut -c1-700
