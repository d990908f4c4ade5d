# Build a variant of libsf_gpu.so with extra defines for sf_fusion.cu (A/B timing):
#   bash tools/variant.sh <name> "-DFOO=1 ..."  -> build/var/<name>/libsf_gpu.so
# Time it with SF_GPU_LIB=build/var/<name>/libsf_gpu.so python tools/integ_time.py
set -e
name=$1; defs=$2
make -s -j8 lib >/dev/null
out=build/var/$name; mkdir -p $out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC,-ffp-contract=off,-O2 -Xptxas -warn-spills $defs -c paper_1311_7194_b200/csrc/sf_fusion.cu -o $out/sf_fusion.o
objs=$(ls build/obj/*.o | grep -v sf_fusion.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libsf_gpu.so $out/sf_fusion.o $objs -Xcompiler -fPIC
echo built $out/libsf_gpu.so
