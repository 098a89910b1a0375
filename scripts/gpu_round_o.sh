python -m paper_2509_21527_b200.build > gpurun_out/o_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/o_pytest1.log 2>&1; echo rc=$? >> gpurun_out/o_pytest1.log
timeout 900 python scripts/overlap.py --config C3 > gpurun_out/o_overlap_C3_n1.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29520 scripts/overlap.py --config C1 > gpurun_out/o_overlap_C1_n2.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 scripts/overlap.py --config C3 > gpurun_out/o_overlap_C3_n2.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 scripts/overlap.py --config C4-1D > gpurun_out/o_overlap_C41D_n2.txt 2>&1
