set -x
L=paper_2509_21527_b200/libhalo.so
timeout 1500 python scripts/ab.py --gpus 2 --libs "rt85=$L@HALO_TREE_ROWS_MAX=85,rt170=$L" --config C4-bw8 --reps 2 --steps 200 > gpurun_out/bw2_ab.txt 2>&1; cut -c1-160 gpurun_out/bw2_ab.txt
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for pr in paper paper_tma auto; do
timeout 600 $R --master-port $((29520 + RANDOM % 400)) bench.py --gpus 2 --config C4-bw8 --no-ns --no-floors --no-e2e --no-graph --no-fused --proto $pr --steps 200 > gpurun_out/bw2_$pr.json 2> gpurun_out/bw2_$pr.err; echo $pr rc=$?
tail -c 300 gpurun_out/bw2_$pr.json | head -c 300; echo
done
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -m gpu -p no:cacheprovider > gpurun_out/bw2_pytest.txt 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/bw2_pytest.txt
