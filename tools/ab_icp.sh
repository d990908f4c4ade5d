for v in "$@"; do echo "== $v"; SF_GPU_LIB=build/var/$v/libsf_gpu.so timeout 300 python tools/icp_time.py 2>&1 | grep -E "steps 1:|steps 2:|all|Error"; done
