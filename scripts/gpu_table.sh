# Round results table: every BASELINE config at 1/2/4 GPUs (+ copy-engine and bandwidth-probe lines).
# Needs a 4-GPU box.  One JSON line per run under gpurun_out/t_<config>_n<N>_<proto>.json
python -m paper_2509_21527_b200.build > gpurun_out/t_build.log 2>&1
run() {  # config gpus proto [extra]
  local c=$1 n=$2 p=$3; shift 3
  if [ "$n" = 1 ]; then
    timeout 600 python bench.py --steps 500 --warmup 20 --config $c --proto $p "$@" > gpurun_out/t_${c}_n${n}_${p}.json 2> gpurun_out/t_${c}_n${n}_${p}.err
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) \
      bench.py --gpus $n --steps 500 --warmup 20 --config $c --proto $p "$@" > gpurun_out/t_${c}_n${n}_${p}.json 2> gpurun_out/t_${c}_n${n}_${p}.err
  fi
}
run C3 1 ll
run C3 1 ce --no-cpu
run C1 1 ll --no-cpu
run C2 1 ll --no-cpu
run C5 1 ll --no-cpu
run C1 2 ll
run C3 2 ll
run C4-1D 2 ll
run C4-1D 2 ce
run C5 2 ll
run C4-bw8 2 ll --no-graph
run C4-bw8 2 ce --no-graph
run C2 4 ll
run C3 4 ll
run C4-2D 4 ll
run C5 4 ll
run C3 4 ce
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/t_reference_C3.json 2> gpurun_out/t_reference_C3.err
# overlap (f1): Alg. 2 skeleton with synthetic NB
timeout 900 python scripts/overlap.py --config C3 > gpurun_out/t_overlap_C3_n1.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29530 scripts/overlap.py --config C1 > gpurun_out/t_overlap_C1_n2.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 scripts/overlap.py --config C3 > gpurun_out/t_overlap_C3_n2.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 scripts/overlap.py --config C4-1D > gpurun_out/t_overlap_C41D_n2.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 scripts/overlap.py --config C2 > gpurun_out/t_overlap_C2_n4.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 scripts/overlap.py --config C4-2D > gpurun_out/t_overlap_C42D_n4.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/t_pytest_mp.log 2>&1; echo rc=$? >> gpurun_out/t_pytest_mp.log
