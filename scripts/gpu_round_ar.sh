python -m paper_2509_21527_b200.build > gpurun_out/ar_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_migrate.py -x -q > gpurun_out/ar_pytest1.log 2>&1; echo rc=$? >> gpurun_out/ar_pytest1.log
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -k "parity" > gpurun_out/ar_pytest2.log 2>&1; echo rc=$? >> gpurun_out/ar_pytest2.log
L=rf=ab/libhalo_rf.so,base=ab/libhalo_cs2.so
python scripts/ab.py --libs $L --config C3 --gpus 1 --reps 3 > gpurun_out/ar_ab_C3_n1.txt 2>&1
python scripts/ab.py --libs $L --config C5 --gpus 1 --reps 3 > gpurun_out/ar_ab_C5_n1.txt 2>&1
python scripts/ab.py --libs $L --config C2 --gpus 1 --reps 2 > gpurun_out/ar_ab_C2_n1.txt 2>&1
python scripts/ab.py --libs $L --config C3 --gpus 2 --reps 2 > gpurun_out/ar_ab_C3_n2.txt 2>&1
python scripts/ab.py --libs $L --config C4-1D --gpus 2 --reps 2 > gpurun_out/ar_ab_C41D_n2.txt 2>&1
python scripts/ab.py --libs $L --config C1 --gpus 2 --reps 2 > gpurun_out/ar_ab_C1_n2.txt 2>&1
timeout 300 python scripts/trace.py --config C3 --flush --queue 10 --no-mid-event > gpurun_out/ar_trace_C3_n1.txt 2>&1
