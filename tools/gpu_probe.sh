set -x
python tools/probe_gemm.py --iters 30 > gpurun_out/probe_gemm.log 2>&1
python tools/probe_gemm.py --iters 30 --linear >> gpurun_out/probe_gemm.log 2>&1
python tools/probe_gemm.py --iters 30 --attention >> gpurun_out/probe_gemm.log 2>&1
cat gpurun_out/probe_gemm.log
