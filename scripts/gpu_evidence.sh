#!/bin/bash
# The standard evidence run on a GPU box (under gpurun, one call):
#   bash scripts/gpu_evidence.sh TAG [NGPUS]
# 1 GPU: GPU test suite, smoke, the default bench line, ncu launch list + one --set full
# capture of the exchange kernels.  N > 1: the test suite (multi-process tests included) and
# the bench line under torchrun (ncu never wraps a multi-rank command).
tag=${1:-ev}; n=${2:-1}; o=gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $o/${tag}_pytest.txt 2>&1; echo pytest_rc=$?
tail -3 $o/${tag}_pytest.txt
if [ "$n" = "1" ]; then
  timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $o/${tag}_smoke.txt 2>&1; echo smoke_rc=$?
  timeout 600 python bench.py > $o/${tag}_bench_n1.json 2> $o/${tag}_bench_n1.err; echo bench_rc=$?
  CMD="python bench.py --steps 20 --warmup 5 --no-cpu --no-graph --no-floors --no-ns --no-fused --no-nccl --no-e2e"
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $o/${tag}_launches.csv $CMD > $o/${tag}_ncu_l.log 2>&1; echo ncu1_rc=$?
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exchange_ll -s 30 -c 2 \
      -o $o/${tag}_ncu_full $CMD > $o/${tag}_ncu_f.log 2>&1; echo ncu2_rc=$?
else
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 29555 bench.py --gpus $n > $o/${tag}_bench_n$n.json 2> $o/${tag}_bench_n$n.err; echo bench_rc=$?
fi
