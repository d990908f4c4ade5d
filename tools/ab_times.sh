# A/B with timelines: integ_time (event timing) + slab_times (per-warp timeline) per variant
for v in "$@"; do echo "== $v"; SF_GPU_LIB=build/var/$v/libsf_gpu.so REPS=${REPS:-2} timeout 300 python tools/integ_time.py 2>&1 | grep -E "us/launch|Error|error"
SF_GPU_LIB=build/var/$v/libsf_gpu.so timeout 300 python tools/slab_times.py 12 codes 2>&1 | grep -E "first|end|Error"; done
