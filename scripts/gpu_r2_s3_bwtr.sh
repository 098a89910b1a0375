set -x
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $R --master-port 29701 scripts/trace.py --config C4-bw8 --flush --queue 3 --no-mid-event > gpurun_out/bwtr.txt 2>&1; echo rc=$?
HALO_DEBUG=8192 timeout 300 $R --master-port 29702 scripts/trace.py --config C4-bw8 --flush --queue 3 --no-mid-event > gpurun_out/bwtr_detail.txt 2>&1; echo rc=$?
grep '^{' gpurun_out/bwtr.txt gpurun_out/bwtr_detail.txt | cut -c1-1500
