set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tnsr.py -x -q 2>&1 | tail -15 > gpurun_out/pytest_tnsr.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
cat gpurun_out/pytest_tnsr.log
