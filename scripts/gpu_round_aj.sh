python -m paper_2509_21527_b200.build > gpurun_out/aj_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ll" > gpurun_out/aj_pytest1.log 2>&1; echo rc=$? >> gpurun_out/aj_pytest1.log
L=t256=ab/libhalo_t256.so,t128=ab/libhalo_t128.so
python scripts/ab.py --libs $L --config C3 --gpus 1 --reps 3 > gpurun_out/aj_ab_C3_n1.txt 2>&1
python scripts/ab.py --libs $L --config C5 --gpus 1 --reps 3 > gpurun_out/aj_ab_C5_n1.txt 2>&1
python scripts/ab.py --libs $L --config C3 --gpus 2 --reps 2 > gpurun_out/aj_ab_C3_n2.txt 2>&1
python scripts/ab.py --libs $L --config C1 --gpus 2 --reps 2 > gpurun_out/aj_ab_C1_n2.txt 2>&1
python scripts/ab.py --libs $L --config C4-1D --gpus 2 --reps 2 > gpurun_out/aj_ab_C41D_n2.txt 2>&1
