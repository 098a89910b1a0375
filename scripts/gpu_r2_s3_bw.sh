set -x
L=paper_2509_21527_b200/libhalo.so
timeout 600 python -m pytest tests/test_gpu_multiproc.py -x -q -m gpu -p no:cacheprovider > gpurun_out/bw_pytest.txt 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/bw_pytest.txt
timeout 1500 python scripts/ab.py --gpus 2 --libs "old=$L@HALO_RING_F=2@HALO_TREE_ROWS_MAX=85,ring4=$L@HALO_TREE_ROWS_MAX=85,new=$L" --config C4-bw8 --reps 2 --steps 200 > gpurun_out/bw_ab.txt 2>&1; cut -c1-140 gpurun_out/bw_ab.txt
timeout 1500 python scripts/ab.py --gpus 2 --libs "old=$L@HALO_RING_F=2@HALO_TREE_ROWS_MAX=85,new=$L" --config C4-1D --reps 2 --steps 200 > gpurun_out/bw_ab_1d.txt 2>&1; cut -c1-140 gpurun_out/bw_ab_1d.txt
