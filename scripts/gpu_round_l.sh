python -m paper_2509_21527_b200.build > gpurun_out/l_build.log 2>&1
L=r64=ab/libhalo_cur.so,r32=ab/libhalo_cur.so@HALO_ITEM_ROWS=32,r128=ab/libhalo_cur.so@HALO_ITEM_ROWS=128,r64l2=ab/libhalo_cur.so+--l2-persist
python scripts/ab.py --libs $L --config C3 --gpus 1 --reps 3 > gpurun_out/l_ab_C3_n1.txt 2>&1
python scripts/ab.py --libs $L --config C3 --gpus 2 --reps 2 > gpurun_out/l_ab_C3_n2.txt 2>&1
python scripts/ab.py --libs $L --config C4-1D --gpus 2 --reps 2 > gpurun_out/l_ab_C41D_n2.txt 2>&1
