timeout 1200 python -m pytest tests/test_gpu_edge_cases.py tests/test_gpu_clique.py -m gpu -x -q > gpurun_out/edge_tests.log 2>&1; tail -n 15 gpurun_out/edge_tests.log
for k in 8 9; do timeout 600 python scripts/ab_clique.py $k build/variants/CP.so paper_2212_04551_b200/libwm_b200.so; done
