"""Per-phase device time of one motif run (WM_PHASES=1) and the gap between
the step's events and the kernel: python scripts/prof_motif_host.py CFG K SUFFIX"""
import os, sys, time
os.environ["WM_PHASES"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_04551_b200 import BalanceConfig, build_dictionary, run_motifs, synth
cfg, k, s = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
g = synth.config_graph(cfg)
d = build_dictionary(k)
lb = BalanceConfig(threshold=1.0, poll_interval=2)
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = run_motifs(g, k, d, mode="opt", balance_config=lb, roots=(g.n - s, g.n))
    torch.cuda.synchronize()
    print("wall %.3f ms  device %.3f ms  kernel %.3f ms" % ((time.perf_counter() - t0) * 1e3,
          r.device_ms, r.kernel_ms), file=sys.stderr, flush=True)
