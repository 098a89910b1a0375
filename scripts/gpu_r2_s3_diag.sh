# diagnostics: set_maps phase profile (C3, 1 GPU), per-CTA traces of the split and the fused step
set -x
HALO_PROFILE=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-graph --no-floors --no-fused --no-nccl > gpurun_out/d_prof.json 2> gpurun_out/d_prof.err; echo rc=$?
grep halo_profile gpurun_out/d_prof.err | tail -12
for i in 1 2; do timeout 120 python scripts/trace.py --config C3 --flush --queue 10 --no-mid-event; done > gpurun_out/d_trace_split.txt 2>&1
timeout 120 python scripts/trace.py --config C3 --flush --queue 10 --fused > gpurun_out/d_trace_fused.txt 2>&1
HALO_DEBUG=8192 timeout 120 python scripts/trace.py --config C3 --flush --queue 10 --no-mid-event > gpurun_out/d_trace_detail.txt 2>&1
cat gpurun_out/d_trace_split.txt gpurun_out/d_trace_fused.txt gpurun_out/d_trace_detail.txt
