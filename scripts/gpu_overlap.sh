# f1 overlap study (Alg. 2 skeleton with synthetic NB) on the final build; needs 4 GPUs
python -m paper_2509_21527_b200.build > gpurun_out/o2_build.log 2>&1
timeout 900 python scripts/overlap.py --config C3 > gpurun_out/o2_overlap_C3_n1.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29530 scripts/overlap.py --config C1 > gpurun_out/o2_overlap_C1_n2.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 scripts/overlap.py --config C3 > gpurun_out/o2_overlap_C3_n2.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 scripts/overlap.py --config C4-1D > gpurun_out/o2_overlap_C41D_n2.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 scripts/overlap.py --config C2 > gpurun_out/o2_overlap_C2_n4.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 scripts/overlap.py --config C4-2D > gpurun_out/o2_overlap_C42D_n4.txt 2>&1
