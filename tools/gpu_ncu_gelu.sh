timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 3 -c 1 -o /tmp/gelu python tools/probe_gemm.py --linear --iters 3 > /dev/null 2>&1
ncu -i /tmp/gelu.ncu-rep --page raw --csv > gpurun_out/raw_gelu.csv 2>/dev/null
ncu -i /tmp/gelu.ncu-rep --page source --csv --print-source sass > gpurun_out/src_gelu.csv 2>/dev/null
ls -la gpurun_out/
