"""Per-phase device times of clique runs (WM_PHASES=1): prof_clique_phases.py CFG K [reps]"""
import os, sys
os.environ["WM_PHASES"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_04551_b200 import BalanceConfig, run_clique, synth
g = synth.config_graph(sys.argv[1])
k = int(sys.argv[2])
bc = BalanceConfig(threshold=1.0, poll_interval=32)
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 3):
    r = run_clique(g, k, mode="opt", balance_config=bc)
    print("count %d kernel %.3f build %.3f device %.3f ms" % (r.clique_count, r.kernel_ms,
          r.extra["build_ms"], r.device_ms), file=sys.stderr, flush=True)
