python -m paper_2509_21527_b200.build > gpurun_out/k_build.log 2>&1
T="scripts/trace.py --config C1 --flush --no-mid-event --steps 10 --queue 10 --no-fshift"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 $T > gpurun_out/k_trace_base.txt 2>&1
HALO_DEBUG=256 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 $T > gpurun_out/k_trace_sink.txt 2>&1
HALO_POLL_NS=200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29516 $T > gpurun_out/k_trace_poll200.txt 2>&1
HALO_DEBUG=256 python scripts/trace.py --config C3 --flush --no-mid-event --steps 10 --queue 10 --no-fshift > gpurun_out/k_trace_C3n1_sink.txt 2>&1
python scripts/trace.py --config C3 --flush --no-mid-event --steps 10 --queue 10 --no-fshift > gpurun_out/k_trace_C3n1_base.txt 2>&1
