timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" 2>&1 | tail -15
timeout 300 python tools/probe_gemm.py --attention --iters 20 2>&1 | tail -3
