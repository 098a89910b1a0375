python -m paper_2509_21527_b200.build > gpurun_out/s_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ll" > gpurun_out/s_pytest1.log 2>&1; echo rc=$? >> gpurun_out/s_pytest1.log
L=tbo=ab/libhalo_tbo.so,tma=ab/libhalo_tma.so,red=ab/libhalo_red.so
python scripts/ab.py --libs $L --config C3 --gpus 1 --reps 3 > gpurun_out/s_ab_C3_n1.txt 2>&1
python scripts/ab.py --libs $L --config C1 --gpus 2 --reps 3 > gpurun_out/s_ab_C1_n2.txt 2>&1
python scripts/ab.py --libs $L --config C4-1D --gpus 2 --reps 2 > gpurun_out/s_ab_C41D_n2.txt 2>&1
HALO_LIB_PATH=ab/libhalo_tbo.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29740 scripts/overlap.py --config C4-1D --protos ll > gpurun_out/s_overlap_C41D_tbo.txt 2>&1
HALO_LIB_PATH=ab/libhalo_tbo.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29741 scripts/overlap.py --config C3 --protos ll > gpurun_out/s_overlap_C3n2_tbo.txt 2>&1
