# Round-end GPU check: parity suite, smoke, bench (N=1), ncu launch list, compute-sanitizer passes.
# usage: bash tools/round_check.sh <tag>   -> gpurun_out/<tag>_*.log / .csv
t=${1:-r2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${t}_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${t}_gputests.log 2>&1; tail -2 gpurun_out/${t}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${t}_smoke.log 2>&1; tail -1 gpurun_out/${t}_smoke.log
timeout 900 python bench.py --steps 60 --warmup 5 > gpurun_out/${t}_bench.log 2>&1; tail -1 gpurun_out/${t}_bench.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${t}_bench_ref.log 2>&1; tail -1 gpurun_out/${t}_bench_ref.log | cut -c1-300
SF_ICP_DEVICE_LOOP=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${t}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5 > gpurun_out/${t}_launches.log 2>&1; tail -c 300 gpurun_out/${t}_launches.log
bash tools/sanitize.sh
