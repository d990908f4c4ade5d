# ncu --set full of the integrate kernel (11th C4 bench frame, plain fuse_frame launches)
# usage: bash tools/ncu_integ.sh <name> <codes|float2> [kernel-regex]
k=${3:-k_integrate_}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 10 --launch-count 1 \
  -o gpurun_out/$1 python tools/integ_profile.py 12 $2 > gpurun_out/$1.log 2>&1; tail -1 gpurun_out/$1.log
