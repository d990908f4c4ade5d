for v in "$@"; do echo "== $v"; SF_GPU_LIB=build/var/$v/libsf_gpu.so timeout 300 python tools/ray_profile.py 12 20 2>&1 | grep -E "raycast:|Error"; done
