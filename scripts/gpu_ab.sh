for lib in M0 MH; do for k in 4 5 6; do WM_B200_LIB=$PWD/build/variants/$lib.so timeout 300 python scripts/var_motif.py cfg2 $k 10; done; done
