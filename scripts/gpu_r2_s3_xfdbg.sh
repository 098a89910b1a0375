set -x
for v in "" "HALO_TREE_ROWS_MAX=85"; do
env $v HALO_COLLAPSE=0 timeout 300 python bench.py --config C4-2D --steps 50 --warmup 5 --no-cpu --no-floors --no-ns --no-e2e --no-graph > gpurun_out/xfdbg.json 2> gpurun_out/xfdbg.err; echo "$v rc=$?"
grep -a "Error" gpurun_out/xfdbg.err | tail -2; tail -c 300 gpurun_out/xfdbg.json; echo
done
HALO_COLLAPSE=0 HALO_ITEM_ROWS=256 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "fused" > gpurun_out/xfdbg_pytest.txt 2>&1; echo rc=$?; tail -3 gpurun_out/xfdbg_pytest.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "fused or int_forces" > gpurun_out/xfdbg_pytest2.txt 2>&1; echo rc=$?; tail -3 gpurun_out/xfdbg_pytest2.txt
