python -m paper_2509_21527_b200.build > gpurun_out/ag_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > gpurun_out/ag_pytest1.log 2>&1; echo rc=$? >> gpurun_out/ag_pytest1.log
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -k "parity" > gpurun_out/ag_pytest2.log 2>&1; echo rc=$? >> gpurun_out/ag_pytest2.log
L=cs=ab/libhalo_cs.so,dx=ab/libhalo_dx.so
python scripts/ab.py --libs $L --config C3 --gpus 1 --reps 3 > gpurun_out/ag_ab_C3_n1.txt 2>&1
python scripts/ab.py --libs $L --config C5 --gpus 1 --reps 3 > gpurun_out/ag_ab_C5_n1.txt 2>&1
python scripts/ab.py --libs $L --config C3 --gpus 2 --reps 2 > gpurun_out/ag_ab_C3_n2.txt 2>&1
python scripts/ab.py --libs $L --config C1 --gpus 2 --reps 2 > gpurun_out/ag_ab_C1_n2.txt 2>&1
