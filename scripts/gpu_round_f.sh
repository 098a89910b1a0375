python -m paper_2509_21527_b200.build > gpurun_out/f_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/f_pytest1.log 2>&1; echo rc=$? >> gpurun_out/f_pytest1.log
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/f_pytest2.log 2>&1; echo rc=$? >> gpurun_out/f_pytest2.log
L=pf=ab/libhalo_pf.so,prev=ab/libhalo_new.so,base=ab/libhalo_r568.so
python scripts/ab.py --libs $L --config C3 --gpus 1 --reps 3 > gpurun_out/f_ab_C3_n1.txt 2>&1
python scripts/ab.py --libs $L --config C1 --gpus 2 --reps 3 > gpurun_out/f_ab_C1_n2.txt 2>&1
python scripts/ab.py --libs $L --config C3 --gpus 2 --reps 2 > gpurun_out/f_ab_C3_n2.txt 2>&1
python scripts/ab.py --libs $L --config C4-1D --gpus 2 --reps 2 > gpurun_out/f_ab_C41D_n2.txt 2>&1
python scripts/ab.py --libs pf=ab/libhalo_pf.so,prev=ab/libhalo_new.so --config C4-bw8 --gpus 2 --reps 2 > gpurun_out/f_ab_C4bw8_n2.txt 2>&1
python scripts/trace.py --config C3 --flush --no-mid-event --steps 10 --queue 10 > gpurun_out/e_trace_C3_n1.txt 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 scripts/trace.py --config C1 --flush --no-mid-event --steps 10 --queue 10 > gpurun_out/e_trace_C1_n2.txt 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 scripts/trace.py --config C4-1D --flush --no-mid-event --steps 10 --queue 10 > gpurun_out/e_trace_C41D_n2.txt 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 scripts/trace.py --config C3 --flush --no-mid-event --steps 10 --queue 10 > gpurun_out/e_trace_C3_n2.txt 2>&1
