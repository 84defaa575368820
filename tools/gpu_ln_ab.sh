mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "layer_norm or ln or step" 2>&1 | tail -3
for i in 1 2; do timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-max-batch 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['value'], d['e2e']['value'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 600 --csv --log-file gpurun_out/launches_warm_ln.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-max-batch > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_warm_ln.csv | head -12
