# GEMM bring-up: tile-variant parity first (bounded), then timings
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "tile_variants or linear or dact or batch_matmul or matmul_t or attention" 2>&1 | tail -25
timeout 300 python tools/probe_gemm.py --iters 30 --sweep 2>&1 | tee gpurun_out/sweep.log
timeout 300 python tools/probe_gemm.py --iters 30 --linear 2>&1 | tee -a gpurun_out/probe_gemm.log
