python -m paper_2509_21527_b200.build > gpurun_out/ai_build.log 2>&1
L=cs2=ab/libhalo_cs2.so,lb4=ab/libhalo_lb4.so,r32=ab/libhalo_cs2.so@HALO_ITEM_ROWS=32,r128=ab/libhalo_cs2.so@HALO_ITEM_ROWS=128
python scripts/ab.py --libs $L --config C3 --gpus 1 --reps 3 > gpurun_out/ai_ab_C3_n1.txt 2>&1
python scripts/ab.py --libs $L --config C5 --gpus 1 --reps 2 > gpurun_out/ai_ab_C5_n1.txt 2>&1
python scripts/ab.py --libs $L --config C3 --gpus 2 --reps 2 > gpurun_out/ai_ab_C3_n2.txt 2>&1
python scripts/ab.py --libs $L --config C1 --gpus 2 --reps 2 > gpurun_out/ai_ab_C1_n2.txt 2>&1
