WM_B200_LIB=$PWD/build/variants/CN.so timeout 900 python -m pytest tests/test_gpu_clique.py tests/test_gpu_edge_cases.py -m gpu -x -q 2>&1 | tail -n 2
for k in 8 7 9 5; do timeout 600 python scripts/ab_clique.py $k build/variants/CP.so build/variants/CN.so; done
