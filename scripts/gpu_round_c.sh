python -m paper_2509_21527_b200.build > gpurun_out/c_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/c_pytest1.log 2>&1; echo rc=$? >> gpurun_out/c_pytest1.log
L=new=ab/libhalo_new.so,base=ab/libhalo_r568.so
python scripts/ab.py --libs $L --config C3 --gpus 1 --reps 3 > gpurun_out/c_ab_C3_n1.txt 2>&1
python scripts/ab.py --libs $L --config C1 --gpus 2 --reps 3 > gpurun_out/c_ab_C1_n2.txt 2>&1
python scripts/ab.py --libs $L --config C4-1D --gpus 2 --reps 2 > gpurun_out/c_ab_C41D_n2.txt 2>&1
python scripts/ab.py --libs $L --config C4-bw8 --gpus 2 --reps 2 > gpurun_out/c_ab_C4bw8_n2.txt 2>&1
python scripts/ab.py --libs new=ab/libhalo_new.so --proto ce --config C4-bw8 --gpus 2 --reps 1 > gpurun_out/c_ab_C4bw8_ce.txt 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 200 --warmup 20 --config C4-bw8 --no-graph > gpurun_out/c_bench_bw8.json 2> gpurun_out/c_bench_bw8.err
