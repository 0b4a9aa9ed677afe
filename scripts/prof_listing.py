"""Warm listing run for ncu capture: prof_listing.py CFG K."""
import sys
sys.path.insert(0, "/root/repo")
from paper_2212_04551_b200 import engine, listing_checksum, synth
engine.LISTING_RING = 1 << 22
g = synth.config_graph(sys.argv[1])
for _ in range(2):
    r = listing_checksum(g, int(sys.argv[2]))
print(r.records_emitted, r.kernel_ms)
