# One ncu --set full capture per top kernel of the C4 bench (SF_ICP_DEVICE_LOOP=0: ncu cannot
# profile kernels inside conditional graph nodes), plus the cold and warm launch lists.
tag=$1
for k in k_integrate_rows k_ray_bounds "k_raycast<" k_raycast_refine k_icp_step; do
  name=$(echo $k | tr -d '<')
  SF_ICP_DEVICE_LOOP=0 timeout 600 ncu --set full --import-source on --clock-control none -k "regex:$k" --launch-skip 6 -c 1 -o gpurun_out/${tag}_$name python bench.py --steps 4 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
SF_ICP_DEVICE_LOOP=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${tag}_launches_cold.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
SF_ICP_DEVICE_LOOP=0 SF_BENCH_NO_FLUSH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 3000 --csv --log-file gpurun_out/${tag}_launches_warm.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out | grep $tag
