python -m paper_2509_21527_b200.build > gpurun_out/u_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > gpurun_out/u_pytest1.log 2>&1; echo rc=$? >> gpurun_out/u_pytest1.log
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/u_pytest2.log 2>&1; echo rc=$? >> gpurun_out/u_pytest2.log
L=head=ab/libhalo_head.so,red=ab/libhalo_red.so,sv2=ab/libhalo_sv2.so,sv2t=ab/libhalo_sv2.so@HALO_POLL_NS=-1
python scripts/ab.py --libs $L --config C3 --gpus 1 --reps 3 > gpurun_out/u_ab_C3_n1.txt 2>&1
python scripts/ab.py --libs $L --config C1 --gpus 2 --reps 3 > gpurun_out/u_ab_C1_n2.txt 2>&1
python scripts/ab.py --libs $L --config C3 --gpus 2 --reps 2 > gpurun_out/u_ab_C3_n2.txt 2>&1
python scripts/ab.py --libs $L --config C4-1D --gpus 2 --reps 2 > gpurun_out/u_ab_C41D_n2.txt 2>&1
