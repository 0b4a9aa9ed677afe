WM_B200_LIB=$PWD/build/variants/CR.so timeout 900 python -m pytest tests/test_gpu_clique.py tests/test_gpu_edge_cases.py -m gpu -x -q 2>&1 | tail -n 2
for k in 8 7 9; do timeout 600 python scripts/ab_clique.py $k build/variants/CP.so build/variants/CR.so; done
WM_B200_LIB=$PWD/build/variants/MS64.so timeout 900 python -m pytest tests/test_gpu_motif.py tests/test_gpu_listing.py -m gpu -x -q 2>&1 | tail -n 2
V="build/variants/M2.so build/variants/MS64.so"
export WM_THR=1.0 WM_POLL=2
timeout 600 python scripts/ab_motif.py cfg4 5 16384 $V
timeout 900 python scripts/ab_motif.py cfg5 7 32768 $V
timeout 600 python scripts/ab_motif.py cfg2 6 0 $V
