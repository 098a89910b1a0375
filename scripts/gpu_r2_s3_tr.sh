set -x
for i in 1 2 3; do
HALO_LIB_PATH=ab/libhalo_head.so timeout 120 python scripts/trace.py --config C3 --flush --queue 10 --no-mid-event > gpurun_out/t_head_$i.txt 2>&1
timeout 120 python scripts/trace.py --config C3 --flush --queue 10 --no-mid-event > gpurun_out/t_new_$i.txt 2>&1
done
cat gpurun_out/t_head_*.txt gpurun_out/t_new_*.txt | cut -c1-900
