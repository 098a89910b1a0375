set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python scripts/trace.py --config C3 --flush --queue 10 > gpurun_out/r2a_trace_C3.txt 2>&1
python bench.py --steps 300 --warmup 20 --no-ns --no-cpu > gpurun_out/r2a_bench_C3.json 2> gpurun_out/r2a_bench_C3.err
tail -c 3000 gpurun_out/r2a_bench_C3.json
cat gpurun_out/r2a_trace_C3.txt
