# Build a variant of libsf_gpu.so with extra defines for some sources (A/B timing):
#   bash tools/variant.sh <name> "-DFOO=1 ..." ["sf_fusion sf_render" (default sf_fusion)]
#   -> build/var/<name>/libsf_gpu.so; time it with SF_GPU_LIB=build/var/<name>/libsf_gpu.so
set -e
IFS=$' \t\n'
name=$1; defs=$2; srcs=${3:-sf_fusion}
if make -s -j8 lib 2>&1 | grep -E "error"; then exit 1; fi
out=build/var/$name; rm -rf "$out"; mkdir -p "$out"
for src in $srcs; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 --expt-relaxed-constexpr \
    -Xcompiler -fPIC,-ffp-contract=off,-O2 $defs -c paper_1311_7194_b200/csrc/$src.cu -o $out/$src.o 2>&1 \
    | grep -v "spill\|^ptxas warning" || true
  test -f $out/$src.o
done
objs=""
for o in build/obj/*.o; do
  b=$(basename $o .o)
  case " $srcs " in *" $b "*) ;; *) objs="$objs $o" ;; esac
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libsf_gpu.so $out/*.o $objs -Xcompiler -fPIC
echo built $out/libsf_gpu.so
