# tests + bench + warm launch list summary (top kernels)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-max-batch 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 600 --csv --log-file gpurun_out/launches_warm.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-max-batch > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_warm.csv > gpurun_out/launches_warm.txt; head -${TOP:-14} gpurun_out/launches_warm.txt
