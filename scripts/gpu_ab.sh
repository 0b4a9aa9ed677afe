WM_B200_LIB=$PWD/build/variants/MK.so python scripts/var_small.py
