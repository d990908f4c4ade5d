# GPU round trip: parity suite, bench (N=1), one ncu capture of a named kernel.
# usage: bash tools/gpu_check.sh <kernel-regex> <launch-skip> <report-name>
timeout 500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
timeout 400 python bench.py --steps 60 --warmup 5 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['stage_ms_mean'], d['roofline']['frac'], d['icp_iterations_mean'])"
if [ -n "$1" ]; then
SF_ICP_DEVICE_LOOP=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:$1 --launch-skip $2 -c 1 -o gpurun_out/$3 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$3.log 2>&1; tail -1 gpurun_out/ncu_$3.log
fi
