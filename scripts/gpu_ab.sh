L=paper_2212_04551_b200/libwm_b200.so
for cfg in "cfg4 5 16384" "cfg5 7 32768" "cfg4 6 65536"; do
for tp in "0.9 8" "1.0 8" "1.0 2" "0.95 4" "1.0 32"; do set -- $tp
echo "thr $1 poll $2: $(WM_THR=$1 WM_POLL=$2 timeout 600 python scripts/ab_motif.py $cfg $L)"
done; done
