"""numpy emulation of the device kernel's data flow over `DeviceLayout`.

Test helper only (CPU tests of the layout maps without a GPU). It walks the
internal block layout exactly the way `csrc/dlmpc.cu` does -- Φ scale per
row from contiguous per-column segments, Ψ per column from the class
operators -- so that, in exact mode, its iterates must be bit-identical to
the oracle's, which proves the index maps before any CUDA runs.
"""

import numpy as np

from oracle.admm_ref import _strict_dot


class LayoutEmulator:
    def __init__(self, L):
        self.L = L
        n = L.n_cols * L.s_pad
        self.psi = np.zeros(n)
        self.lam = np.zeros(n)
        self.psi_prev = np.zeros(n)
        self.lam_prev = np.zeros(n)
        self.s_row = np.zeros(L.n_rows)
        self.x = np.zeros(L.n_cols)
        self.ada = np.zeros(L.n_sub)
        lens = np.diff(L.ball_ptr)
        self.d_row = int(max(L.state_count[L.ball_idx[L.ball_ptr[i]:L.ball_ptr[i + 1]]].sum()
                             for i in range(L.n_sub)))
        self.row_len_sub = np.array([L.state_count[L.ball_idx[L.ball_ptr[i]:L.ball_ptr[i + 1]]].sum()
                                     for i in range(L.n_sub)])

    def _cols_of(self, i):
        L = self.L
        out = []
        for e in range(L.ball_ptr[i], L.ball_ptr[i + 1]):
            j = L.ball_idx[e]
            for c in range(L.state_start[j], L.state_start[j] + L.state_count[j]):
                out.append((c, int(L.ball_off[e])))
        return out

    def set_x(self, x):
        self.x = np.asarray(x, dtype=np.float64).copy()
        for i in range(self.L.n_sub):
            cs = [c for c, _ in self._cols_of(i)]
            v = self.x[cs]
            acc = _strict_dot(v[None, :], v[None, :])[0]
            if len(cs) < self.d_row:
                acc = acc + 0.0
            self.ada[i] = acc

    def phi_scale(self):
        L = self.L
        rho = L.rho
        for i in range(L.n_sub):
            cols = self._cols_of(i)
            r0, r1 = L.row_start[i], L.row_start[i + 1]
            for l in range(r1 - r0):
                pos = np.array([c * L.s_pad + off + l for c, off in cols])
                v = self.psi[pos] - self.lam[pos]
                xs = self.x[[c for c, _ in cols]]
                acc = _strict_dot(v[None, :], xs[None, :])[0]
                if len(cols) < self.d_row:
                    acc = acc + 0.0
                ir = r0 + l
                ada = self.ada[i]
                y0 = rho * acc / (rho + 2.0 * L.row_w[ir] * ada)
                y = min(max(y0, L.row_lo[ir]), L.row_hi[ir])
                self.s_row[ir] = (y - acc) / ada if ada > 0 else 0.0

    def _support_rows(self, j):
        L = self.L
        rows = []
        for e in range(L.ball_ptr[j], L.ball_ptr[j + 1]):
            i = L.ball_idx[e]
            rows.extend(range(L.row_start[i], L.row_start[i + 1]))
        return np.array(rows)

    def phi_internal(self, psi, lam):
        L = self.L
        phi = np.zeros_like(psi)
        for c in range(L.n_cols):
            j = L.col_owner[c]
            S = L.col_len[c]
            sl = slice(c * L.s_pad, c * L.s_pad + S)
            phi[sl] = (psi[sl] - lam[sl]) + self.s_row[self._support_rows(j)] * self.x[c]
        return phi

    def iterate(self):
        L = self.L
        self.phi_scale()
        phi = self.phi_internal(self.psi, self.lam)
        new_psi = np.zeros_like(self.psi)
        new_lam = np.zeros_like(self.lam)
        pri = dual = 0.0
        for c in range(L.n_cols):
            k = L.col_class[c]
            S, m = int(L.class_s[k]), int(L.class_m[k])
            j = L.col_owner[c]
            rp = L.ref_pos[j, :S].astype(np.int64)
            base = c * L.s_pad
            ph = phi[base:base + S]
            lm = self.lam[base:base + S]
            ps = self.psi[base:base + S]
            if L.exact:
                g = L.g_pool[L.class_g_off[k]:L.class_g_off[k + 1]].reshape(m, S)
                P = L.p_pool[L.class_p_off[k]:L.class_p_off[k + 1]].reshape(S, m)
                rhs = L.rhs_pool[L.col_vec[c] * L.m_pad:L.col_vec[c] * L.m_pad + m]
                kref = ph[rp] + lm[rp]
                resid = rhs - (g * kref[None, :]).sum(axis=1)
                pref = kref + (P * resid[None, :]).sum(axis=1)
                pn = np.zeros(S)
                pn[rp] = pref
            else:
                ldn, n0 = int(L.class_ldn[k]), int(L.class_n0[k])
                blk = L.null_pool[L.class_null_off[k]:L.class_null_off[k + 1]].reshape(-1, ldn)
                N = blk[:S, :n0]
                kv = ph + lm
                q = L.q_pool[L.col_vec[c] * L.s_pad:L.col_vec[c] * L.s_pad + S]
                pn = q + N @ (N.T @ kv)
            d = ph - pn
            new_psi[base:base + S] = pn
            new_lam[base:base + S] = lm + d
            pri = max(pri, float(np.max(np.abs(d))))
            dual = max(dual, float(np.max(np.abs(pn - ps))))
        self.psi_prev, self.lam_prev = self.psi, self.lam
        self.psi, self.lam = new_psi, new_lam
        self.phi = phi
        return pri, L.rho * dual
