WM_B200_LIB=$PWD/build/variants/ME.so timeout 900 python -m pytest tests/test_gpu_motif.py tests/test_gpu_listing.py -m gpu -x -q 2>&1 | tail -n 1
WM_B200_LIB=$PWD/build/variants/ME.so timeout 900 python scripts/shard_scaling.py 2>&1 | grep motif | cut -c1-400
