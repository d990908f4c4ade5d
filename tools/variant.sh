# Build a variant of libsf_gpu.so with extra defines for one source (A/B timing):
#   bash tools/variant.sh <name> "-DFOO=1 ..." [source (default sf_fusion)]  -> build/var/<name>/libsf_gpu.so
# Time it with SF_GPU_LIB=build/var/<name>/libsf_gpu.so python tools/integ_time.py
set -e
name=$1; defs=$2; src=${3:-sf_fusion}
make -s -j8 lib >/dev/null 2>&1
out=build/var/$name; mkdir -p $out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC,-ffp-contract=off,-O2 $defs -c paper_1311_7194_b200/csrc/$src.cu -o $out/$src.o 2>&1 | grep -v "spill\|^ptxas warning" || true
objs=$(ls build/obj/*.o | grep -v "/$src.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libsf_gpu.so $out/$src.o $objs -Xcompiler -fPIC
echo built $out/libsf_gpu.so
