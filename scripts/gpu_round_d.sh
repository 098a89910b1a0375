python -m paper_2509_21527_b200.build > gpurun_out/d_build.log 2>&1
python scripts/trace.py --config C3 --flush --no-mid-event --steps 20 > gpurun_out/d_trace_C3_n1.txt 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 scripts/trace.py --config C1 --flush --no-mid-event --steps 20 > gpurun_out/d_trace_C1_n2.txt 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 scripts/trace.py --config C1 --flush --steps 20 > gpurun_out/d_trace_C1_n2_mid.txt 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 scripts/trace.py --config C1 --flush --no-mid-event --no-fshift --steps 20 > gpurun_out/d_trace_C1_n2_nofs.txt 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 scripts/trace.py --config C1 --no-mid-event --steps 20 > gpurun_out/d_trace_C1_n2_noflush.txt 2>&1
