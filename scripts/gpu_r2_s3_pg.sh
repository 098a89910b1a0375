set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "packed or step_host or graph or stale" > gpurun_out/pg_pytest.txt 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pg_pytest.txt
for g in 1 0; do
HALO_PACKED_GRAPH=$g timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu --no-floors --no-ns --no-graph --no-fused > gpurun_out/pg_b_$g.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/pg_b_$g.json').read().strip().splitlines()[-1]); print('graph=$g', d['value'], d['e2e'])"
done
L=paper_2509_21527_b200/libhalo.so
timeout 1200 python scripts/ab.py --libs "xf4=$L,xf3=ab/libhalo_xf3.so" --config C3 --reps 2 > gpurun_out/xf3_ab.txt 2>&1; cut -c1-170 gpurun_out/xf3_ab.txt
