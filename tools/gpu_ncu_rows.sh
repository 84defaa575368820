# one --set full capture per row kernel; only CSV summaries come back
for k in k_ln_fwd k_ln_bwd k_colsum_partial k_attn_fwd k_attn_bwd k_embed_rank; do
  timeout 300 ncu --set full --clock-control none -k regex:$k -s 5 -c 1 -o /tmp/prof_$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /tmp/ncu_$k.log 2>&1
  ncu -i /tmp/prof_$k.ncu-rep --page raw --csv > gpurun_out/raw_$k.csv 2>/dev/null
  ncu -i /tmp/prof_$k.ncu-rep --page details --csv > gpurun_out/details_$k.csv 2>/dev/null
  tail -2 /tmp/ncu_$k.log
done
ls -la gpurun_out
