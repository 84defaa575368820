# alternating whole-step A/B of prebuilt libtcb200.so variants in alt_libs/ (args: variant names)
L=paper_2303_04759_b200/lib/libtcb200.so
for v in "$@"; do cp alt_libs/$v.so $L; timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm" -p no:cacheprovider 2>&1 | tail -1; done
for r in 1 2 3 4; do for v in "$@"; do cp alt_libs/$v.so $L; echo -n "$v "; timeout 300 python tools/ab_cfg.py base 2>/dev/null | head -1; done; done
