# Round-end verification: GPU tests, smoke, both bench arms, launch lists, one ncu --set full of the top GEMM.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_cold.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-max-batch > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_gemm_tc -s 40 -c 1 -o /tmp/gemm_step python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-max-batch > /dev/null 2>&1
ncu -i /tmp/gemm_step.ncu-rep --page raw --csv > gpurun_out/raw_gemm_step.csv 2>/dev/null
ncu -i /tmp/gemm_step.ncu-rep --page details --csv > gpurun_out/details_gemm_step.csv 2>/dev/null
tail -3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log
tail -1 gpurun_out/bench_full.json gpurun_out/bench_ref.json
python tools/launches.py gpurun_out/launches_cold.csv | head -25
