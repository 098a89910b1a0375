python -m paper_2509_21527_b200.build > gpurun_out/ac_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_migrate.py tests/test_gpu_parity.py tests/test_gpu_pme.py -x -q > gpurun_out/ac_pytest1.log 2>&1; echo rc=$? >> gpurun_out/ac_pytest1.log
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -k "migrate or pme" > gpurun_out/ac_pytest2.log 2>&1; echo rc=$? >> gpurun_out/ac_pytest2.log
HALO_PROFILE=1 timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu --no-graph --no-nccl --pme > gpurun_out/ac_bench_C3_n1.json 2> gpurun_out/ac_bench_C3_n1.err
HALO_PROFILE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29861 bench.py --gpus 2 --steps 100 --warmup 10 --config C4-1D --no-cpu --no-graph --no-nccl --pme > gpurun_out/ac_bench_C41D_n2.json 2> gpurun_out/ac_bench_C41D_n2.err
# final-build ncu evidence (1 GPU, C3 = 8 DD ranks)
CMD="python bench.py --steps 20 --warmup 5 --no-cpu --no-graph --no-floors --no-ns --no-nccl"
$CMD > gpurun_out/ac_ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ac_ncu_launches.csv $CMD > gpurun_out/ac_ncu_l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_exchange -s 20 -c 4 -o gpurun_out/ac_ncu_full $CMD > gpurun_out/ac_ncu_f.log 2>&1
echo rc=$? > gpurun_out/ac_ncu_rc.txt
ncu -i gpurun_out/ac_ncu_full.ncu-rep --page raw --csv > gpurun_out/ac_ncu_raw.csv 2>/dev/null
