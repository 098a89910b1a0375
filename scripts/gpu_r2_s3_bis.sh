set -x
L=paper_2509_21527_b200/libhalo.so
timeout 1800 python scripts/ab.py --libs "head=ab/libhalo_head.so,new=$L,nostale=ab/libhalo_nostale.so,nopf=ab/libhalo_nopf.so,noboth=ab/libhalo_noboth.so,nozero=$L@HALO_AB_NO_LLZERO=1,hostplan=$L@HALO_PLAN_HOST=1" --config C3 --reps 3 > gpurun_out/b_ab_C3.txt 2>&1; cut -c1-140 gpurun_out/b_ab_C3.txt
