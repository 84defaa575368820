timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 7 -c 1 -o /tmp/dact python tools/probe_gemm.py --linear --iters 2 > /dev/null 2>&1
ncu -i /tmp/dact.ncu-rep --page raw --csv > gpurun_out/raw_dact.csv 2>/dev/null
ncu -i /tmp/dact.ncu-rep --page source --csv --print-source sass > gpurun_out/src_dact.csv 2>/dev/null
head -c 300 gpurun_out/raw_dact.csv | tail -c 200
