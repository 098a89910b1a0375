# 4 GPUs: hop groups (HEAD) vs the pre-hop-group build (21dfc17) vs HALO_COLLAPSE=0, C3 and C5; fused C4-2D check
set -x
L=paper_2509_21527_b200/libhalo.so
timeout 1500 python scripts/ab.py --gpus 4 --libs "now=$L,pre=ab/libhalo_21dfc17.so,staged=$L@HALO_COLLAPSE=0" --config C3 --reps 2 --steps 200 > gpurun_out/n4ab_C3.txt 2>&1; cut -c1-150 gpurun_out/n4ab_C3.txt
timeout 900 python scripts/ab.py --gpus 4 --libs "now=$L,pre=ab/libhalo_21dfc17.so" --config C5 --reps 2 --steps 200 > gpurun_out/n4ab_C5.txt 2>&1; cut -c1-150 gpurun_out/n4ab_C5.txt
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29613 bench.py --gpus 4 --config C4-2D --no-floors --no-ns > gpurun_out/n4ab_C42D.json 2> gpurun_out/n4ab_C42D.err; echo rc=$?
tail -c 500 gpurun_out/n4ab_C42D.json; grep -a Error gpurun_out/n4ab_C42D.err | tail -3
