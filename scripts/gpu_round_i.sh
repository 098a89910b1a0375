python -m paper_2509_21527_b200.build > gpurun_out/i_build.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29510 scripts/probe_launch.py > gpurun_out/i_probe.txt 2>&1
L=cur=ab/libhalo_cur.so,fence=ab/libhalo_cur.so@HALO_DEBUG=128,nopdl=ab/libhalo_cur.so@HALO_PDL=0
python scripts/ab.py --libs $L --config C1 --gpus 2 --reps 2 > gpurun_out/i_ab_C1_n2.txt 2>&1
python scripts/ab.py --libs $L --config C3 --gpus 2 --reps 2 > gpurun_out/i_ab_C3_n2.txt 2>&1
python scripts/ab.py --libs $L --config C3 --gpus 1 --reps 2 > gpurun_out/i_ab_C3_n1.txt 2>&1
