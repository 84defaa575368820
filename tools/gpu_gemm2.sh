timeout 300 python tools/probe_gemm.py --iters 30 --sweep 2>&1 | tee gpurun_out/sweep.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 3 -c 1 -o gpurun_out/prof_gelu python tools/probe_gemm.py --linear --iters 3 > gpurun_out/ncu_gelu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 3 -c 1 -o gpurun_out/prof_ffn1 python tools/probe_gemm.py --only 2 --iters 3 > gpurun_out/ncu_ffn1.log 2>&1
ls -la gpurun_out
