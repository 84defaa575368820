timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "multicast" 2>&1 | tail -5
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "tile_variants or split_k" 2>&1 | tail -2
timeout 600 python tools/probe_gemm.py --iters 20 --sweep 2>&1 | tee gpurun_out/sweep_mc.log
