set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "int_forces or fused or graph" > gpurun_out/r128_pytest.txt 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/r128_pytest.txt
HALO_ITEM_ROWS=128 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "int_forces or fused" > gpurun_out/r128_pytest2.txt 2>&1; echo pytest2_rc=$?; tail -2 gpurun_out/r128_pytest2.txt
for rep in 1 2; do
for r in 64 128; do
HALO_ITEM_ROWS=$r timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu --no-floors --no-ns --no-e2e --no-graph > gpurun_out/r128_b_${r}_$rep.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/r128_b_${r}_$rep.json').read().strip().splitlines()[-1]); print('R=$r', d['value'], d['x_us'], d['f_us'], d['fused_xf']['us_per_step'])"
done; done
