for j in 4 8 16 32 64; do SF_RAY_JUMP_CELLS=$j timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$j', round(d['value']), d['stage_ms_mean']['raycast'])"; done
timeout 500 python -m pytest tests -m gpu -x -q -k "ray or tracker or golden" 2>&1 | tail -1
