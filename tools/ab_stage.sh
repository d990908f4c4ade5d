# A/B of the tracked frame's stage times (in-graph events): raycast, icp, fuse prologue, integrate, total (us)
for v in "$@"; do echo "== $v"; SF_GPU_LIB=build/var/$v/libsf_gpu.so STAGES=2 timeout 300 python tools/icp_time.py 2>&1 | grep -E "^all|Error"; done
