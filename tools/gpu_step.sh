timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
TCB_PDL=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PDL=0', d['value'], d['ms_per_step'])"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PDL=1', d['value'], d['ms_per_step'])"
