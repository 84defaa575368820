timeout 300 python tools/probe_gemm.py --trace 2>&1 | tee gpurun_out/trace.log
