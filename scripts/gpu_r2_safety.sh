export HALO_G3_LOG=gpurun_out/r2b_g3.jsonl
rm -f $HALO_G3_LOG
timeout 1500 python -m pytest tests/test_gpu_safety.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r2b_safety.txt 2>&1
tail -30 gpurun_out/r2b_safety.txt
cat $HALO_G3_LOG
