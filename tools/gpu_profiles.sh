# Round profile refresh: full bench JSON, launch list (cold = ncu default, and warm), one --set full capture of the
# top GEMM from the bench step (CSV summaries only come back).
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
tail -1 gpurun_out/bench_full.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_cold.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-max-batch > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 600 --csv --log-file gpurun_out/launches_warm.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-max-batch > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_gemm_tc -s 40 -c 1 -o /tmp/gemm_step python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-max-batch > /dev/null 2>&1
ncu -i /tmp/gemm_step.ncu-rep --page raw --csv > gpurun_out/raw_gemm_step.csv 2>/dev/null
ncu -i /tmp/gemm_step.ncu-rep --page details --csv > gpurun_out/details_gemm_step.csv 2>/dev/null
python tools/launches.py gpurun_out/launches_warm.csv | head -25
