timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "split_k or tile_variants" 2>&1 | tail -5
timeout 300 python tools/probe_gemm.py --iters 20 --splits 2>&1 | tee gpurun_out/splits.log
