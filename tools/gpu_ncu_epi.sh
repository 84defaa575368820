# --set full of the GELU forward (launch 1), the act=deriv dgrad (launch 3) and the plain GEMM (launch 5)
for i in 1 3 5; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s $i -c 1 -o /tmp/epi$i python tools/ncu_epi.py > /dev/null 2>&1
  ncu -i /tmp/epi$i.ncu-rep --page raw --csv > gpurun_out/raw_epi$i.csv 2>/dev/null
  ncu -i /tmp/epi$i.ncu-rep --page source --csv --print-source sass > gpurun_out/src_epi$i.csv 2>/dev/null
done
ls gpurun_out | head
