# A/B/C clique variants (build/variants/*.so), cfg3 at k=7,8,9
for k in 8 7 9; do timeout 600 python scripts/ab_clique.py $k build/variants/A.so build/variants/B.so build/variants/C.so; done
