# One ncu --set full capture per top kernel of the C4 bench at a late frame (launch-skip 40 of
# the 60-step run: ~22 k blocks, the bench's mean), plus the cold and warm launch lists of the
# whole run. SF_ICP_DEVICE_LOOP=0: ncu cannot profile kernels inside conditional graph nodes.
tag=$1
for k in k_integrate_rows k_ray_bounds "k_raycast<" k_raycast_refine k_icp_step; do
  name=$(echo $k | tr -d '<')
  SF_ICP_DEVICE_LOOP=0 timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$k" --launch-skip 40 -c 1 -o gpurun_out/${tag}_$name python bench.py --steps 60 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
done
SF_ICP_DEVICE_LOOP=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file gpurun_out/${tag}_launches_cold.csv python bench.py --steps 60 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
SF_ICP_DEVICE_LOOP=0 SF_BENCH_NO_FLUSH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 12000 --csv --log-file gpurun_out/${tag}_launches_warm.csv python bench.py --steps 60 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out | grep $tag
