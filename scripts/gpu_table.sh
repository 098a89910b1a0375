# Round results table: every BASELINE config at 1/2/4 GPUs (+ transports, zones, PME, bandwidth probes).
# Needs a 4-GPU box.  One JSON line per run under gpurun_out/t_<config>_n<N>_<tag>.json
python -m paper_2509_21527_b200.build > gpurun_out/t_build.log 2>&1
run() {  # config gpus tag [bench args]
  local c=$1 n=$2 t=$3; shift 3
  if [ "$n" = 1 ]; then
    timeout 600 python bench.py --steps 500 --warmup 20 --config $c "$@" > gpurun_out/t_${c}_n${n}_${t}.json 2> gpurun_out/t_${c}_n${n}_${t}.err
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) \
      bench.py --gpus $n --steps 500 --warmup 20 --config $c "$@" > gpurun_out/t_${c}_n${n}_${t}.json 2> gpurun_out/t_${c}_n${n}_${t}.err
  fi
}
run C3 1 ll --pme
run C3 1 ce --proto ce --no-cpu --no-ns
run C3 1 rounded --zones rounded --no-cpu --no-ns
run C1 1 ll --no-cpu
run C2 1 ll --no-cpu
run C5 1 ll --no-cpu
run C1 2 ll --no-cpu
run C1 2 paper --proto paper --no-cpu --no-ns
run C1 2 paper_tma --proto paper_tma --no-cpu --no-ns
run C3 2 ll --no-cpu
run C4-1D 2 ll --no-cpu --pme
run C4-1D 2 ce --proto ce --no-cpu --no-ns
run C4-1D 2 paper --proto paper --no-cpu --no-ns
run C4-1D 2 paper_tma --proto paper_tma --no-cpu --no-ns
run C5 2 ll --no-cpu
run C4-bw5 2 ll --no-graph --no-cpu --no-ns
run C4-bw5 2 ce --proto ce --no-graph --no-cpu --no-ns
run C4-bw8 2 ll --no-graph --no-cpu --no-ns
run C4-bw8 2 ce --proto ce --no-graph --no-cpu --no-ns
run C4-bw8 2 auto --proto auto --no-graph --no-cpu --no-ns
run C2 4 ll --no-cpu
run C3 4 ll --no-cpu --pme
run C3 4 rounded --zones rounded --no-cpu --no-ns
run C4-2D 4 ll --no-cpu
run C5 4 ll --no-cpu
run C3 4 ce --proto ce --no-cpu --no-ns
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/t_reference_C3.json 2> gpurun_out/t_reference_C3.err
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/t_pytest_mp.log 2>&1; echo rc=$? >> gpurun_out/t_pytest_mp.log
timeout 1200 python -m pytest tests -m gpu -x -q --ignore=tests/test_gpu_multiproc.py > gpurun_out/t_pytest_all.log 2>&1; echo rc=$? >> gpurun_out/t_pytest_all.log
# final-build ncu evidence (1 GPU, C3 = 8 DD ranks)
CMD="python bench.py --steps 20 --warmup 5 --no-cpu --no-graph --no-floors --no-ns --no-nccl"
$CMD > gpurun_out/t_ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/t_ncu_launches.csv $CMD > gpurun_out/t_ncu_l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_exchange -s 20 -c 4 -o gpurun_out/t_ncu_full $CMD > gpurun_out/t_ncu_f.log 2>&1
echo rc=$? > gpurun_out/t_ncu_rc.txt
ncu -i gpurun_out/t_ncu_full.ncu-rep --page raw --csv > gpurun_out/t_ncu_raw.csv 2>/dev/null
