# GPU-scope LL loads/stores (valid only when every peer is on this GPU): N = 1 only
L=sys=ab/libhalo_final.so,gpu=ab/libhalo_gpuscope.so
python scripts/ab.py --libs $L --config C3 --gpus 1 --reps 3 > gpurun_out/at_ab_C3_n1.txt 2>&1
python scripts/ab.py --libs $L --config C5 --gpus 1 --reps 3 > gpurun_out/at_ab_C5_n1.txt 2>&1
python scripts/ab.py --libs $L --config C2 --gpus 1 --reps 3 > gpurun_out/at_ab_C2_n1.txt 2>&1
python scripts/ab.py --libs $L --config C1 --gpus 1 --reps 3 > gpurun_out/at_ab_C1_n1.txt 2>&1
