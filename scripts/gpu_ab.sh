for k in 8 7 9; do timeout 600 python scripts/ab_clique.py $k build/variants/CDa.so build/variants/CD65536.so build/variants/C4.so; done
