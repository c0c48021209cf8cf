"""Graph partition of the DLMPC hot path across GPUs.

Rank r owns a contiguous range of subsystems (its columns). One ADMM
iteration on rank r needs:

* the Φ scale of every row its columns touch: the *patch* P_r, the union of
  the closed d-hop balls of its own subsystems;
* for those rows, ψ and λ of every column in their supports: the columns of
  H_r = union of the balls of P_r (2d hops). The *halo* H_r minus own is
  received from the ranks owning it, once per iteration, after they finish
  their Ψ/Λ stage;
* the global maximum of the (pri, dual) residuals: an all-reduce(max) of two
  doubles, which is also the only global synchronisation.

Per MPC step the measured state x is needed on H_r (row data, control,
plant step couple at most 2d hops). Per-entry arithmetic does not depend on
the partition, so a k-GPU run is bit-identical to the 1-GPU run (the C5
parity test, SURVEY §8(e) "Determinism").

This module only plans the exchange; `tests/test_multirank.py` runs the
partitioned iteration on CPU ranks (gloo, world size 2) against the
single-domain iteration.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class RankPlan:
    rank: int
    own: tuple                 # [lo, hi) subsystems
    patch: np.ndarray          # subsystems whose rows need a Φ scale
    need: np.ndarray           # subsystems whose columns are read (own + halo)
    recv: dict                 # source rank -> halo subsystems received each iteration
    send: dict                 # destination rank -> own subsystems sent each iteration


def _ball_union(ball_ptr, ball_idx, subs):
    if len(subs) == 0:
        return np.zeros(0, dtype=np.int64)
    return np.unique(np.concatenate([ball_idx[ball_ptr[i]:ball_ptr[i + 1]] for i in subs]))


def plan_partition(mask, world: int, weights=None):
    """Contiguous, column-balanced subsystem ranges per rank and the halo
    exchange lists between them."""
    cm = mask.compact
    if cm is None:
        raise ValueError("partitioning needs a mask built by build_locality_mask")
    n = int(cm["state_start"].size)
    if world < 1 or world > n:
        raise ValueError("world size must be between 1 and the number of subsystems")
    cols = np.asarray(cm["state_count"] if weights is None else weights, dtype=np.float64)
    cum = np.concatenate([[0.0], np.cumsum(cols)])
    cuts = [0] + [int(np.searchsorted(cum, cum[-1] * r / world)) for r in range(1, world)] + [n]
    for r in range(1, world + 1):          # non-empty ranges
        cuts[r] = max(cuts[r], cuts[r - 1] + 1)
    cuts[world] = n
    owner = np.empty(n, dtype=np.int64)
    for r in range(world):
        owner[cuts[r]:cuts[r + 1]] = r
    ptr, idx = cm["ball_ptr"], cm["ball_idx"].astype(np.int64)
    plans = []
    for r in range(world):
        own = np.arange(cuts[r], cuts[r + 1])
        patch = _ball_union(ptr, idx, own)
        need = _ball_union(ptr, idx, patch)
        halo = need[(need < cuts[r]) | (need >= cuts[r + 1])]
        recv = {}
        for q in np.unique(owner[halo]):
            recv[int(q)] = halo[owner[halo] == q]
        plans.append(RankPlan(r, (cuts[r], cuts[r + 1]), patch, need, recv, {}))
    for p in plans:
        for q, subs in p.recv.items():
            plans[q].send[p.rank] = subs
    return plans


def halo_bytes_per_iteration(plans, mask, s_pad):
    """Bytes each rank receives per ADMM iteration (ψ and λ, full columns)."""
    cnt = mask.compact["state_count"]
    return [int(sum(cnt[subs].sum() for subs in p.recv.values())) * s_pad * 2 * 8 for p in plans]
