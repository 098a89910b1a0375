python -m paper_2509_21527_b200.build > gpurun_out/h_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/h_pytest1.log 2>&1; echo rc=$? >> gpurun_out/h_pytest1.log
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/h_pytest2.log 2>&1; echo rc=$? >> gpurun_out/h_pytest2.log
L=cur=ab/libhalo_cur.so,l2=ab/libhalo_cur.so+--l2-persist,pf=ab/libhalo_pf.so
python scripts/ab.py --libs $L --config C3 --gpus 1 --reps 3 > gpurun_out/h_ab_C3_n1.txt 2>&1
python scripts/ab.py --libs $L --config C1 --gpus 2 --reps 3 > gpurun_out/h_ab_C1_n2.txt 2>&1
python scripts/ab.py --libs $L --config C4-1D --gpus 2 --reps 2 > gpurun_out/h_ab_C41D_n2.txt 2>&1
python bench.py --steps 500 --warmup 20 > gpurun_out/h_bench_C3_n1.json 2> gpurun_out/h_bench_C3_n1.err
