import sys, json
sys.path.insert(0, "/root/repo")
from paper_2212_04551_b200 import BalanceConfig, run_clique, synth
g = synth.config_graph("cfg3")
bc = BalanceConfig(threshold=1.0, poll_interval=32)
def show(tag, **kw):
    rs = [run_clique(g, 9, **kw) for _ in range(4)]
    r = rs[-1]
    print(tag, json.dumps({"kernel_ms": round(r.kernel_ms, 3), "device_ms": round(r.device_ms, 3),
          "idle": round(r.idle_warp_fraction, 3), "tasks": r.tasks, "count": r.clique_count,
          "warps": r.warps, "migr": r.migrations, "don": r.rebalance_count}), flush=True)
show("tiny-roots-opt", mode="opt", balance_config=bc, order="id", roots=(99990, 100000))
show("shard64-opt", mode="opt", balance_config=bc, shard=(5, 64), reduce=False)
show("shard64-wc", mode="wc", shard=(5, 64), reduce=False)
show("full-opt", mode="opt", balance_config=bc)
show("shard64-opt-warps1", mode="opt", balance_config=bc, shard=(5, 64), reduce=False, blocks_per_sm=1)
show("full-opt-bps2", mode="opt", balance_config=bc, blocks_per_sm=2)
show("full-opt-bps3", mode="opt", balance_config=bc, blocks_per_sm=3)
