# A/B: time the integrate kernel for each variant library under build/var/<name>
for v in "$@"; do echo "== $v"; SF_GPU_LIB=build/var/$v/libsf_gpu.so REPS=${REPS:-2} timeout 300 python tools/integ_time.py 2>&1 | grep -E "us/launch|Error|error" ; done
