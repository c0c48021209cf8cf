"""numpy restatement of the reference DLMPC ADMM iteration (the checker).

TEST INFRASTRUCTURE ONLY -- see `oracle/__init__.py`. Each stage cites the
reference lines it restates; the arithmetic order is the reference's:

* Φ row stage      admm.py:155-170, ascending_dot sls_core.py:37-47
* Φ row->col copy  sls_core.py:442-446
* Ψ column stage   admm.py:174-186 (numpy pairwise `.sum(axis=-1)` over the
                   reference support order; columns batched by shape, which
                   never changes a column's own reduction, admm.py:77-94)
* Λ update         admm.py:205-207
* residuals        admm.py:214-217, 269-270
* Ψ/Λ col->row     sls_core.py:448-456
* solve loop       admm.py:315-347
* u extraction     admm.py:350-360
* plant step       admm.py:363-369
* closed loop      admm.py:437-540 (recurring phases only)

Inputs are the host-side setup objects (LayoutTables, ColumnPrecomp list,
RowData), which the test-suite pins bit-for-bit against the reference's own
objects (`tests/test_setup_parity.py`). `workers > 1` shards the row and
column stages over a thread pool the way the reference's `fused` schedule
does (strategies.py:195-206, 301-306); results are identical for any worker
count because no item's arithmetic depends on the batch.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np


def _strict_dot(x, y):
    acc = np.multiply(x[..., 0], y[..., 0])
    for j in range(1, x.shape[-1]):
        acc = np.add(acc, np.multiply(x[..., j], y[..., j]))
    return acc


class OracleSolver:
    """Reference-order ADMM on the dual padded layout (one session)."""

    def __init__(self, tables, col_solvers, rho, workers=1):
        self.t = tables
        self.rho = float(rho)
        self.workers = max(1, int(workers))
        self.pool = ThreadPoolExecutor(self.workers) if self.workers > 1 else None
        n_r, d_r, n_c, d_c = tables.n_rows, tables.d_row, tables.n_cols, tables.d_col
        self.phi_r = np.zeros((n_r, d_r)); self.psi_r = np.zeros((n_r, d_r)); self.lam_r = np.zeros((n_r, d_r))
        self.phi_c = np.zeros((n_c, d_c)); self.psi_c = np.zeros((n_c, d_c)); self.lam_c = np.zeros((n_c, d_c))
        self.psi_prev_c = np.zeros((n_c, d_c))
        self.pri_c = np.zeros(n_c); self.dual_c = np.zeros(n_c)
        # group columns by operator shape; stack their operators once. Columns
        # whose precomps share ONE g / projector object (the class-built
        # list of precompute_column_solvers) keep a single broadcast copy:
        # the (cols x m x s) product is still materialised before the
        # pairwise sum, so each column's reduction is unchanged, and N=10^4
        # needs 0.5 MB instead of 10 GB of operators.
        groups = {}
        for c, pre in enumerate(col_solvers):
            groups.setdefault((pre.g.shape, id(pre.g), id(pre.projector)), []).append(c)
        shared = len(groups) < len(col_solvers) // 2
        if not shared:
            groups = {}
            for c, pre in enumerate(col_solvers):
                groups.setdefault((pre.g.shape, 0, 0), []).append(c)
        self.groups = []
        for key in sorted(groups, key=lambda k: (k[0], groups[k][0])):
            cols = np.asarray(groups[key], dtype=np.int64)
            n = key[0][1]
            if shared:
                g = col_solvers[cols[0]].g[None]
                P = col_solvers[cols[0]].projector[None]
            else:
                g = np.stack([col_solvers[c].g for c in cols])
                P = np.stack([col_solvers[c].projector for c in cols])
            self.groups.append(dict(
                cols=cols, shared=shared, g=g, P=P,
                rhs=np.stack([col_solvers[c].rhs for c in cols]),
                cells=cols[:, None] * d_c + np.arange(n)[None, :]))
        self.row_data = None
        self._phi_src = np.where(tables.col_valid, tables.c2r_flat, 0)
        self._row_src = np.where(tables.row_valid, tables.r2c_flat, 0)

    def close(self):
        if self.pool is not None:
            self.pool.shutdown()
            self.pool = None

    def zero_(self):
        for a in (self.phi_r, self.psi_r, self.lam_r, self.phi_c, self.psi_c, self.lam_c,
                  self.psi_prev_c):
            a.fill(0.0)

    def _shards(self, n):
        if self.pool is None or n < 2 * self.workers:
            return [(0, n)]
        step = -(-n // self.workers)
        return [(lo, min(lo + step, n)) for lo in range(0, n, step)]

    def _run(self, n, body):
        shards = self._shards(n)
        if len(shards) == 1:
            body(*shards[0])
        else:
            for f in [self.pool.submit(body, lo, hi) for lo, hi in shards]:
                f.result()

    # -- stages -----------------------------------------------------------------
    def _phi(self, lo, hi):
        rd = self.row_data
        v = self.psi_r[lo:hi] - self.lam_r[lo:hi]
        a = rd.a_pad[lo:hi]
        ada = rd.a_dot_a[lo:hi]
        c = _strict_dot(v, a)
        y0 = self.rho * c / (self.rho + 2.0 * rd.weight[lo:hi] * ada)
        y = np.clip(y0, rd.lo[lo:hi], rd.hi[lo:hi])
        scale = np.where(ada > 0.0, (y - c) / np.where(ada > 0.0, ada, 1.0), 0.0)
        self.phi_r[lo:hi] = v + scale[:, None] * a

    def _psi_block(self, grp, i0, i1):
        phi, lam = self.phi_c.ravel(), self.lam_c.ravel()
        psi, prev = self.psi_c.ravel(), self.psi_prev_c.ravel()
        cells = grp["cells"][i0:i1]
        k = phi[cells] + lam[cells]
        g = grp["g"] if grp["shared"] else grp["g"][i0:i1]
        P = grp["P"] if grp["shared"] else grp["P"][i0:i1]
        resid = grp["rhs"][i0:i1] - (g * k[:, None, :]).sum(axis=2)
        prev[cells] = psi[cells]
        psi[cells] = k + (P * resid[:, None, :]).sum(axis=2)

    def _cols(self, lo, hi):
        for grp in self.groups:
            # a group's columns are ascending but need not be contiguous
            i0 = int(np.searchsorted(grp["cols"], lo))
            i1 = int(np.searchsorted(grp["cols"], hi))
            # small chunks keep the (cols x m x s) product temporaries in cache
            for j0 in range(i0, i1, 8):
                self._psi_block(grp, j0, min(j0 + 8, i1))
        self.lam_c[lo:hi] += self.phi_c[lo:hi] - self.psi_c[lo:hi]
        self.pri_c[lo:hi] = np.abs(self.phi_c[lo:hi] - self.psi_c[lo:hi]).max(axis=-1)
        self.dual_c[lo:hi] = self.rho * np.abs(self.psi_c[lo:hi] - self.psi_prev_c[lo:hi]).max(axis=-1)

    def iterate(self):
        """One ADMM iteration; returns the reduced (pri, dual)."""
        t = self.t
        self._run(t.n_rows, self._phi)
        vals = self.phi_r.ravel()[self._phi_src]
        vals[~t.col_valid] = 0.0
        self.phi_c[:] = vals
        # Groups hold sorted, disjoint column ids; shard ranges of columns.
        self._run(t.n_cols, self._cols)
        vals = self.psi_c.ravel()[self._row_src]
        vals[~t.row_valid] = 0.0
        self.psi_r[:] = vals
        vals = self.lam_c.ravel()[self._row_src]
        vals[~t.row_valid] = 0.0
        self.lam_r[:] = vals
        return float(self.pri_c.max()), float(self.dual_c.max())

    def iterate_sequential(self):
        """One iteration in the reference's `sequential` schedule
        (strategies.py:262-281, the paper's single-thread "CPU ADMM"): every
        stage called one row / one column at a time, stage after stage, on
        one core. Same arithmetic as `iterate` (batching never changes an
        item's reduction, admm.py:6-10); only the per-item call structure --
        which is where that schedule's time goes -- differs."""
        t = self.t
        if not hasattr(self, "_col_slot"):
            self._col_slot = {}
            for grp in self.groups:
                for i, c in enumerate(grp["cols"]):
                    self._col_slot[int(c)] = (grp, i)
        for r in range(t.n_rows):
            self._phi(r, r + 1)
        vals = self.phi_r.ravel()[self._phi_src]
        vals[~t.col_valid] = 0.0
        self.phi_c[:] = vals
        for c in range(t.n_cols):
            grp, i = self._col_slot[c]
            self._psi_block(grp, i, i + 1)
        for c in range(t.n_cols):
            self.lam_c[c:c + 1] += self.phi_c[c:c + 1] - self.psi_c[c:c + 1]
        for c in range(t.n_cols):
            self.pri_c[c:c + 1] = np.abs(self.phi_c[c:c + 1] - self.psi_c[c:c + 1]).max(axis=-1)
            self.dual_c[c:c + 1] = self.rho * np.abs(self.psi_c[c:c + 1] - self.psi_prev_c[c:c + 1]).max(axis=-1)
        vals = self.psi_c.ravel()[self._row_src]
        vals[~t.row_valid] = 0.0
        self.psi_r[:] = vals
        vals = self.lam_c.ravel()[self._row_src]
        vals[~t.row_valid] = 0.0
        self.lam_r[:] = vals
        return float(self.pri_c.max()), float(self.dual_c.max())

    def solve(self, row_data, max_iters, eps_pri, eps_dual, sequential=False):
        """admm.py:315-347: returns (iterations, history, converged)."""
        self.row_data = row_data
        hist = []
        step = self.iterate_sequential if sequential else self.iterate
        for _ in range(max_iters):
            pri, dual = step()
            hist.append((pri, dual))
            if pri <= eps_pri and dual <= eps_dual:
                return len(hist), hist, True
        return len(hist), hist, False


def row_data_for(x, tables, weight, lo, hi):
    """sls_core.py:330-349 without the per-row Python loop: (a_pad, ada) plus
    the first infeasible row or -1."""
    a_pad = np.where(tables.row_valid, x[tables.rs_safe], 0.0)
    ada = _strict_dot(a_pad, a_pad)
    bad = np.nonzero((ada == 0.0) & ((lo > 0.0) | (hi < 0.0)))[0]

    class _RD:
        pass
    rd = _RD()
    rd.a_pad, rd.a_dot_a, rd.weight, rd.lo, rd.hi = a_pad, ada, weight, lo, hi
    return rd, (int(bad[0]) if bad.size else -1)


def extract_control(phi_r, tables, x, input_rows):
    """admm.py:350-360: u_k = ascending dot of φ_r[r_k] with x on the support."""
    u = np.zeros(len(input_rows))
    for k, r in enumerate(input_rows):
        n = int(tables.row_len[r])
        u[k] = float(_strict_dot(phi_r[r, :n], x[tables.rs[r, :n]]))
    return u


def step_dynamics(a, b, x, u):
    """admm.py:363-369 (scipy CSR mat-vecs)."""
    return a @ x + b @ u


def simulate(system, spec, tables, col_solvers, x0, t_sim, warm_start=True, workers=1,
             solver=None, sequential=False):
    """Closed loop of admm.py:437-540 (recurring phases). Returns dict with
    states, inputs, step_iterations, histories; raises nothing -- failures are
    reported as `status` ('ok' | 'not_converged' | 'row_infeasible') + `step`."""
    weight, lo, hi = spec.row_arrays()
    n_x, t = system.n_states, spec.horizon
    input_rows = [n_x * t + k for k in range(system.n_inputs)]
    own = solver is None
    if own:
        solver = OracleSolver(tables, col_solvers, spec.rho, workers)
    else:
        solver.zero_()
    x = np.asarray(x0, dtype=np.float64)
    states, inputs, iters, hists = [x], [], [], []
    status, at = "ok", None
    try:
        for step in range(t_sim):
            rd, bad = row_data_for(x, tables, weight, lo, hi)
            if bad >= 0:
                status, at = "row_infeasible", (step, bad)
                break
            if not warm_start:
                solver.zero_()
            n_it, hist, ok = solver.solve(rd, spec.max_iters, spec.eps_pri, spec.eps_dual, sequential)
            hists.append(hist)
            if not ok:
                status, at = "not_converged", (step, None)
                break
            iters.append(n_it)
            u = extract_control(solver.phi_r, tables, x, input_rows)
            x = step_dynamics(system.a, system.b, x, u)
            inputs.append(u)
            states.append(x)
    finally:
        if own:
            solver.close()
    return dict(states=np.array(states), inputs=np.array(inputs).reshape(len(inputs), system.n_inputs),
                step_iterations=iters, histories=hists, status=status, at=at, solver=solver)
