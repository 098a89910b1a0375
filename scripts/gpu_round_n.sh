python -m paper_2509_21527_b200.build > gpurun_out/n_build.log 2>&1
L=bo=ab/libhalo_bo.so,red=ab/libhalo_red.so,bocap2=ab/libhalo_bo.so@HALO_CTAS_PER_SM=2
python scripts/ab.py --libs $L --config C3 --gpus 1 --reps 2 > gpurun_out/n_ab_C3_n1.txt 2>&1
python scripts/ab.py --libs $L --config C1 --gpus 2 --reps 2 > gpurun_out/n_ab_C1_n2.txt 2>&1
python scripts/ab.py --libs $L --config C4-1D --gpus 2 --reps 2 > gpurun_out/n_ab_C41D_n2.txt 2>&1
for v in "red ab/libhalo_red.so 0" "bo ab/libhalo_bo.so 0" "bocap2 ab/libhalo_bo.so 2" "bocap1 ab/libhalo_bo.so 1"; do
  set -- $v
  HALO_LIB_PATH=$2 HALO_CTAS_PER_SM=$3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) scripts/overlap.py --config C4-1D --protos ll > gpurun_out/n_overlap_C41D_$1.txt 2>&1
  HALO_LIB_PATH=$2 HALO_CTAS_PER_SM=$3 timeout 600 python scripts/overlap.py --config C3 --protos ll > gpurun_out/n_overlap_C3n1_$1.txt 2>&1
done
