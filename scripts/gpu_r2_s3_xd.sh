set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "fused or tag_wrap or stale" > gpurun_out/xd_pytest.txt 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/xd_pytest.txt
for rep in 1 2; do
timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu --no-floors --no-ns --no-e2e --no-graph > gpurun_out/xd_b_$rep.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/xd_b_$rep.json').read().strip().splitlines()[-1]); print('C3', d['value'], d['x_us'], d['f_us'], d['fused_xf'].get('us_per_step'), d['fused_xf'].get('median_us'))"
done
timeout 120 python scripts/trace.py --config C3 --flush --queue 10 --fused > gpurun_out/xd_trace.txt 2>&1; grep '^{' gpurun_out/xd_trace.txt | cut -c1-900
