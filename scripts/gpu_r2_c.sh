export HALO_G3_LOG=gpurun_out/r2c_g3.jsonl
rm -f $HALO_G3_LOG
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "fused" > gpurun_out/r2c_fused.txt 2>&1
tail -5 gpurun_out/r2c_fused.txt
timeout 300 python bench.py --steps 300 --warmup 20 --no-ns --no-cpu --no-floors > gpurun_out/r2c_bench_C3.json 2> gpurun_out/r2c_bench_C3.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2c_bench_C3.json").read())
print("value", d["value"], "graph", d["graph_us_per_step"], "fused", d["fused_xf"], "x", d["x_us"], "f", d["f_us"])
PY
tail -3 gpurun_out/r2c_bench_C3.err
timeout 900 python -m pytest tests/test_gpu_safety.py -q -m gpu -p no:cacheprovider > gpurun_out/r2c_safety.txt 2>&1
tail -5 gpurun_out/r2c_safety.txt
cat $HALO_G3_LOG
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r2c_parity.txt 2>&1
tail -5 gpurun_out/r2c_parity.txt
