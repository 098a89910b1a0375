python -m paper_2509_21527_b200.build > gpurun_out/j_build.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29510 scripts/probe_launch.py > gpurun_out/j_probe.txt 2>&1
HALO_PDL=0 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 scripts/trace.py --config C1 --flush --no-mid-event --steps 10 --queue 10 > gpurun_out/j_trace_C1_n2_nopdl.txt 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 scripts/trace.py --config C1 --flush --no-mid-event --steps 10 --queue 10 > gpurun_out/j_trace_C1_n2.txt 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 scripts/trace.py --config C1 --no-mid-event --steps 10 --queue 10 > gpurun_out/j_trace_C1_n2_noflush.txt 2>&1
