"""Dense KKT reference solve for unbounded instances -- TEST INFRASTRUCTURE ONLY.

Restates the reference's secondary ground truth
(`/root/reference/pkg/src/locality_mpc/oracle.py:25-108` kkt_oracle_equality,
111-127 simulate_with_oracle): with all bounds infinite, the horizon problem
is an equality-constrained least-squares problem in the stacked support
entries of every column,

    min  sum_r w_r (phi_r . x)^2   s.t.  g0_c z_c = rhs0_c  for every column c,

solved directly through its KKT system with `lstsq` (the cost may be
singular on the feasible set). It shares nothing with the ADMM iteration
except the problem statement, which is what makes agreement meaningful
(the reference's acceptance test compares closed-loop costs at 1e-4,
test_acceptance.py:112-132). Limited to small instances (dense system).
"""

from __future__ import annotations

import numpy as np

MAX_SUPPORT_ENTRIES = 6000   # reference oracle.py:22


def kkt_response(system, spec, mask, x):
    """Dense (n_rows, n_cols) response minimising the quadratic row costs at
    state x subject to the locality-restricted dynamics constraints."""
    from paper_2103_14990_b200 import build_dynamics_operator, row_index_map
    x = np.asarray(x, dtype=np.float64)
    if mask.n_entries > MAX_SUPPORT_ENTRIES:
        raise ValueError("instance too large for the dense KKT oracle")
    metas = row_index_map(system.partition, spec.horizon, spec)
    if any(np.isfinite(m.lo) or np.isfinite(m.hi) for m in metas):
        raise ValueError("the equality oracle requires all bounds infinite")
    op = build_dynamics_operator(system, spec.horizon)
    z_csc = op.z.tocsc()
    sups = [np.asarray(s, dtype=np.int64) for s in mask.col_supports]
    offs = np.concatenate([[0], np.cumsum([s.size for s in sups])]).astype(np.int64)
    n = int(offs[-1])
    # position of (row, column) in the stacked vector
    pos = {}
    for c, s in enumerate(sups):
        for j, r in enumerate(s.tolist()):
            pos[(r, c)] = int(offs[c] + j)
    h = np.zeros((n, n))
    for r, sup in enumerate(mask.row_supports):
        w = metas[r].weight
        if w == 0.0:
            continue
        idx = np.array([pos[(r, int(c))] for c in sup])
        vec = np.zeros(n)
        vec[idx] = x[np.asarray(sup, dtype=np.int64)]
        h += 2.0 * w * np.outer(vec, vec)
    blocks = []
    for c, s in enumerate(sups):
        sub = z_csc[:, s]
        touch = np.unique(sub.tocoo().row)
        blocks.append((np.asarray(sub.toarray()[touch]), (touch == c).astype(np.float64)))
    m = sum(g.shape[0] for g, _ in blocks)
    kkt = np.zeros((n + m, n + m))
    rhs = np.zeros(n + m)
    kkt[:n, :n] = h
    row = n
    for c, (g, r0) in enumerate(blocks):
        k = g.shape[0]
        kkt[row:row + k, offs[c]:offs[c + 1]] = g
        kkt[offs[c]:offs[c + 1], row:row + k] = g.T
        rhs[row:row + k] = r0
        row += k
    sol = np.linalg.lstsq(kkt, rhs, rcond=None)[0]
    z = sol[:n]
    feas = float(np.max(np.abs(kkt[n:, :n] @ z - rhs[n:])))
    if feas > 1e-8 * max(1.0, float(np.max(np.abs(rhs)))):
        raise RuntimeError(f"KKT solve violates the constraints ({feas:.3e})")
    dense = np.zeros((mask.n_rows, mask.n_cols))
    for c, s in enumerate(sups):
        dense[s, c] = z[offs[c]:offs[c + 1]]
    return dense


def kkt_closed_loop(system, spec, mask, x0, t_sim):
    """Closed loop driven by the dense KKT solve (reference oracle.py:111-127).
    Returns (states, inputs)."""
    n_x, t = system.n_states, spec.horizon
    x = np.asarray(x0, dtype=np.float64)
    states, inputs = [x], []
    for _ in range(t_sim):
        dense = kkt_response(system, spec, mask, x)
        u = np.array([float(dense[n_x * t + k] @ x) for k in range(system.n_inputs)])
        x = system.a @ x + system.b @ u
        inputs.append(u)
        states.append(x)
    return np.array(states), np.array(inputs)
