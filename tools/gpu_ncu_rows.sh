# --set full captures of the row / memory-bound kernels of the bench step (CSV exports come back)
for k in ${KERNELS:-k_ln_fwd16 k_ln_bwd16 k_ln_colsum k_colsum_partial k_adam k_attn_fwd k_attn_bwd}; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 5 -c 1 -o /tmp/prof_$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-max-batch > /tmp/ncu_$k.log 2>&1
  ncu -i /tmp/prof_$k.ncu-rep --page raw --csv > gpurun_out/raw_$k.csv 2>/dev/null
  ncu -i /tmp/prof_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$k.csv 2>/dev/null
done
ls -la gpurun_out | head -30
