# ncu evidence for the current build (1 GPU, C3 = 8 DD ranks): launch list + --set full of the exchange kernels
set -x
CMD="python bench.py --steps 20 --warmup 5 --no-cpu --no-graph --no-floors --no-ns --no-fused"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_launches.csv $CMD > gpurun_out/ncu_l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_exchange -s 20 -c 4 -o gpurun_out/ncu_full $CMD > gpurun_out/ncu_f.log 2>&1
echo rc=$?
