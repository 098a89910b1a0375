# PDL overlap: steady-state traces without the mid event, x grid capped to leave room for f CTAs
set -x
for cap in 0 4 3 2; do
  if [ $cap = 0 ]; then unset HALO_X_CTAS_PER_SM; else export HALO_X_CTAS_PER_SM=$cap; fi
  timeout 120 python scripts/trace.py --config C3 --flush --queue 10 --no-mid-event > gpurun_out/pdl_trace_$cap.txt 2>&1
  timeout 300 python bench.py --steps 500 --no-ns --no-cpu --no-floors --no-graph --no-fused > gpurun_out/pdl_bench_$cap.json 2> gpurun_out/pdl_bench_$cap.err
done
