# ncu --set full of the three raycast kernels (plain sf_raycast launches on a C4 volume)
# usage: bash tools/ncu_ray.sh <name>
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_ray_bounds|k_raycast" --launch-skip 9 --launch-count 3 \
  -o gpurun_out/$1 python tools/ray_profile.py 12 3 > gpurun_out/$1.log 2>&1; tail -1 gpurun_out/$1.log
