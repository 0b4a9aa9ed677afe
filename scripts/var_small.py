"""Small-graph motif timing variance vs resident warps and GPU warm state:
python scripts/var_small.py"""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2212_04551_b200 import BalanceConfig, build_dictionary, run_motifs, run_clique, synth
g = synth.config_graph("cfg2")
d = build_dictionary(4)
bc = BalanceConfig(threshold=0.9, poll_interval=8)
for bps in (0, 2, 1):
    ms = []
    for i in range(8):
        r = run_motifs(g, 4, d, mode="opt", balance_config=bc, blocks_per_sm=bps)
        ms.append(round(r.kernel_ms, 3))
    print("bps", bps, "warps", r.warps, "idle %.3f" % r.idle_warp_fraction, ms, flush=True)
# with the GPU kept busy just before each run (clock ramp)
x = torch.randn(4096, 4096, device="cuda")
ms = []
for i in range(8):
    for _ in range(20):
        x = x @ x
        x /= x.norm()
    r = run_motifs(g, 4, d, mode="opt", balance_config=bc)
    ms.append(round(r.kernel_ms, 3))
print("busy-before", "warps", r.warps, ms, flush=True)
ms = []
for i in range(8):
    r = run_motifs(g, 4, d, mode="wc")
    ms.append(round(r.kernel_ms, 3))
print("wc", "warps", r.warps, ms, flush=True)
