"""Where the e2e step's time goes beyond the device step (host-side phases)."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
from paper_2212_04551_b200 import BalanceConfig, engine, run_clique, synth
from paper_2212_04551_b200.graph import CsrGraph
g = synth.config_graph("cfg3")
bc = BalanceConfig(threshold=1.0, poll_interval=32)
s = torch.cuda.current_stream()
off_h = torch.from_numpy(np.array(g.offsets)).pin_memory()
nbr_h = torch.from_numpy(np.array(g.neighbors_array)).pin_memory()
for _ in range(3):
    run_clique(g, 8, mode="opt", balance_config=bc, stream=s, reduce=False)
for it in range(5):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    gh = CsrGraph(g.n, off_h.numpy(), nbr_h.numpy()); t.append(time.perf_counter())
    engine.device_graph(gh); torch.cuda.synchronize(); t.append(time.perf_counter())
    r = run_clique(gh, 8, mode="opt", balance_config=bc, stream=s, reduce=False)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    engine.release_device_graph(gh); torch.cuda.synchronize(); t.append(time.perf_counter())
    r2 = run_clique(g, 8, mode="opt", balance_config=bc, stream=s, reduce=False)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
    print("ctor %.3f create+upload %.3f run %.3f (device_ms %.3f kernel %.3f) release %.3f | warm run %.3f (device_ms %.3f)"
          % (d[0], d[1], d[2], r.device_ms, r.kernel_ms, d[3], d[4], r2.device_ms), flush=True)
