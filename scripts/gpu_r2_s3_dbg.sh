set -x
HALO_PROFILE=1 timeout 300 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize.py --case T3D --protos ll > gpurun_out/dbg_memcheck.txt 2>&1; echo rc=$?
head -80 gpurun_out/dbg_memcheck.txt
