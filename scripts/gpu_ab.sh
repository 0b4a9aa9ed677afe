WM_B200_LIB=$PWD/build/variants/MWD.so timeout 900 python -m pytest tests/test_gpu_motif.py tests/test_gpu_listing.py -m gpu -x -q 2>&1 | tail -n 1
V="build/variants/MWD.so build/variants/MW256.so"
export WM_THR=1.0 WM_POLL=2
timeout 600 python scripts/ab_motif.py cfg4 5 16384 $V
timeout 900 python scripts/ab_motif.py cfg5 7 32768 $V
timeout 600 python scripts/ab_motif.py cfg5 5 65536 $V
timeout 600 python scripts/ab_motif.py cfg2 6 0 $V
