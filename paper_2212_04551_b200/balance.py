"""Load-balancing configuration (reference ``pkg/src/warpmine/balance.py``).

The reference's Coordinator (``balance.py:163-194``) runs on the host between
scheduler rounds: poll active warps, stop everyone at a consistent state,
steal the shallowest pending extension for each idle warp round-robin, resume.
On B200 the same policy runs on the device inside the enumeration kernel
(``csrc/wm_common.cuh`` ``acquire_work`` / ``donation_wanted`` and the donation
blocks of ``wm_clique.cu`` / ``wm_motif.cu``): idle warps register on a global
counter, and busy warps poll it every ``poll_interval`` DFS steps and donate
their shallowest pending extension through a bounded device queue — no
kernel stop/relaunch.  ``BalanceConfig`` keeps the reference's knobs and
validation so ``run(..., balance_config=...)`` calls are unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass

ACTIVE = "active"
IDLE = "idle"
STOPPED = "stopped"

CLIQUE_THRESHOLD = 0.40
MOTIF_THRESHOLD = 0.10
DEFAULT_POLL_INTERVAL = 10


@dataclass(frozen=True)
class BalanceConfig:
    """threshold: donate when active/total warps falls below it.
    poll_interval: DFS steps between a busy warp's idle-counter polls.
    (reference ``balance.py:36-52``)"""

    threshold: float = CLIQUE_THRESHOLD
    poll_interval: int = DEFAULT_POLL_INTERVAL
    enabled: bool = True

    def __post_init__(self):
        if not 0.0 < self.threshold <= 1.0:
            raise ValueError("threshold must be in (0, 1]")
        if self.poll_interval < 1:
            raise ValueError("poll_interval must be >= 1")


def default_config(app_name: str) -> BalanceConfig:
    """Per-application defaults (reference ``balance.py:55-60``)."""
    if app_name == "clique":
        return BalanceConfig(threshold=CLIQUE_THRESHOLD)
    return BalanceConfig(threshold=MOTIF_THRESHOLD)


def should_rebalance(active: int, total: int, cfg: BalanceConfig) -> bool:
    """Host restatement of the trigger the device evaluates
    (reference ``balance.py:63-66``)."""
    if total <= 0:
        raise ValueError("total warp count must be positive")
    return active / total < cfg.threshold
