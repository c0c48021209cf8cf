"""Device data layout of the DLMPC hot path (built once per session, on host).

The reference keeps every iterate twice -- padded row-major (n_rows x d_row)
and padded column-major (n_cols x d_col) -- and copies between the two
layouts every iteration (sls_core.py:352-472). The device keeps ONE copy:

* **Internal row order**: rows grouped by owning subsystem, ascending
  reference index inside a subsystem (`row_start`, `int_to_ref`).
* **Block column layout**: column c (owner j) stores its support as the
  concatenation over ball members i of j (ascending) of the rows of i, padded
  to `s_pad` doubles (a multiple of 4 >= d_col: the paper's longest-vector
  padding). Entry (row of i with local index l, column c) sits at
  `c*s_pad + ball_off[e(i->j)] + l`. A row's neighbourhood is therefore a set
  of contiguous per-column segments (coalesced Φ-stage reads), and a column
  is one contiguous vector (coalesced Ψ-stage tiles). The Ψ/Λ col->row
  exchange disappears: the Φ stage reads this layout directly.
* **Column classes**: columns whose reference operator `g0` is bit-identical
  and whose support permutation agrees share one device class. The fast path
  stores an orthonormal null-space basis N of each class (internal order,
  zero padded to [round8(s)][ldn], ldn = 4 mod 16 so that the FP64 MMA
  fragment loads are bank-conflict free) and one particular solution q per
  distinct (class, rhs); Ψ = q + N(Nᵀ k) is the reference projection
  k + P(rhs - g k) (admm.py:186) in exact arithmetic. The exact path stores
  the reference's own g, P (reference support order) and reduced rhs.
* **Tiles**: columns sorted by class, cut into tiles of `tile_cols` (8/16)
  columns; one CTA works a tile at a time.
"""

from __future__ import annotations

import numpy as np

from .sls_core import ColumnClasses, ProblemSpec
from .system_model import LocalityMask, LtiSystem

SM_COUNT_B200 = 148


def _round(n, m):
    return ((int(n) + m - 1) // m) * m


def _ld_frag(n):
    """Smallest leading dimension >= n with ld % 16 in (4, 12): conflict-free
    8x4 / 4x8 FP64 fragment loads (a half-warp's 4 rows of 4 consecutive
    doubles land on 16 distinct 8-byte banks)."""
    ld = max(int(n), 1)
    while ld % 16 not in (4, 12):
        ld += 1
    return ld


def choose_tile_cols(n_cols, sm_count=SM_COUNT_B200):
    """Largest tile that still gives every SM work; >= 8 (one MMA n-tile)."""
    for tc in (16,):
        if n_cols >= 2 * tc * sm_count:
            return tc
    return 8


class DeviceLayout:
    """All arrays of `dlmpc_problem` (include/dlmpc.h) plus the index maps
    between the internal layout and the reference's padded layouts."""

    def __init__(self, system: LtiSystem | None, spec: ProblemSpec, mask: LocalityMask,
                 classes: ColumnClasses, exact: bool = False, tile_cols: int | None = None,
                 own=None):
        if mask.compact is None:
            raise ValueError("the device layout needs a mask built by build_locality_mask")
        cm = mask.compact
        t = int(spec.horizon)
        if cm["horizon"] != t:
            raise ValueError("mask horizon does not match the spec")
        self.exact = bool(exact)
        self.rho = float(spec.rho)
        n_sub = int(cm["state_start"].size)
        n_x, n_u = int(cm["n_x"]), int(cm["n_u"])
        self.n_sub, self.n_cols, self.n_inputs, self.horizon = n_sub, n_x, n_u, t
        # owned subsystem range (graph partition); the rest is a read-only halo
        own = (0, n_sub) if own is None else (int(own[0]), int(own[1]))
        self.own_sub = own
        st0 = cm["state_start"]
        self.own_cols = (int(st0[own[0]]), int(st0[own[1] - 1] + cm["state_count"][own[1] - 1]))
        s_cnt, u_cnt = cm["state_count"], cm["input_count"]
        rows_per = cm["rows_per_sub"]
        self.n_rows = int(rows_per.sum())
        self.row_start = np.concatenate([[0], np.cumsum(rows_per)]).astype(np.int64)

        # internal <-> reference row order
        owner_ref = cm["row_owner"].astype(np.int64)
        self.int_to_ref = np.argsort(owner_ref, kind="stable").astype(np.int64)
        self.ref_to_int = np.empty_like(self.int_to_ref)
        self.ref_to_int[self.int_to_ref] = np.arange(self.n_rows)
        self.row_owner_int = owner_ref[self.int_to_ref]
        local_of_ref = self.ref_to_int - self.row_start[owner_ref]

        # balls and block offsets
        ball_ptr, ball_idx = cm["ball_ptr"], cm["ball_idx"].astype(np.int64)
        deg = np.diff(ball_ptr)
        src = np.repeat(np.arange(n_sub, dtype=np.int64), deg)
        r_of = rows_per[ball_idx]
        excl = np.cumsum(r_of) - r_of
        excl -= np.repeat(excl[ball_ptr[:-1]] if ball_idx.size else np.zeros(0, np.int64), deg)
        # excl[e'] with e' = (j -> i): offset of i's block inside j's support.
        key_e = src * n_sub + ball_idx            # CSR order == sorted
        key_t = ball_idx * n_sub + src            # the transposed pair
        order_t = np.argsort(key_t, kind="stable")
        if not np.array_equal(key_t[order_t], key_e):
            raise ValueError("balls are not symmetric")
        self.ball_ptr = ball_ptr.astype(np.int64)
        self.ball_idx = ball_idx.astype(np.int32)
        self.ball_off = excl[order_t].astype(np.int32)   # for e = (i -> j): offset of i in j
        self._key_e = key_e
        sup_len = np.add.reduceat(r_of, ball_ptr[:-1]) if ball_idx.size else np.zeros(n_sub, np.int64)
        self.col_len_sub = sup_len.astype(np.int64)
        self.s_pad = _round(int(sup_len.max()), 4)
        gaps = np.diff(ball_idx)
        row_bound = np.zeros(ball_idx.size, dtype=bool)
        row_bound[ball_ptr[:-1][deg > 0]] = True
        self.contiguous = bool(np.all(gaps[~row_bound[1:]] == 1)) if ball_idx.size > 1 else True
        self.state_start = cm["state_start"].astype(np.int32)
        self.state_count = s_cnt.astype(np.int32)
        # row-support descriptor per subsystem: (column, block offset) pairs in
        # ascending column order -- the reference's ascending_dot order.
        cnt_e = s_cnt[ball_idx]
        self.supp_len = np.add.reduceat(cnt_e, ball_ptr[:-1]).astype(np.int32)
        self.d_pad = _round(int(self.supp_len.max()), 4)
        e_rep = np.repeat(np.arange(ball_idx.size), cnt_e)
        k_in_e = np.arange(e_rep.size) - np.repeat(np.cumsum(cnt_e) - cnt_e, cnt_e)
        sub_of = src[e_rep]
        first_of_sub = np.cumsum(np.r_[0, self.supp_len[:-1].astype(np.int64)])
        slot = np.arange(e_rep.size) - first_of_sub[sub_of]
        self.supp_col = np.zeros((n_sub, self.d_pad), dtype=np.int32)
        self.supp_off = np.zeros((n_sub, self.d_pad), dtype=np.int32)
        self.supp_col[sub_of, slot] = (cm["state_start"][ball_idx[e_rep]] + k_in_e).astype(np.int32)
        self.supp_off[sub_of, slot] = self.ball_off[e_rep]

        # per-row costs and bounds, internal order
        w, lo, hi = spec.row_arrays()
        self.row_w = np.ascontiguousarray(w[self.int_to_ref])
        self.row_lo = np.ascontiguousarray(lo[self.int_to_ref])
        self.row_hi = np.ascontiguousarray(hi[self.int_to_ref])
        excl_zero = (self.row_lo > 0.0) | (self.row_hi < 0.0)
        first_bad = np.full(n_sub, -1, dtype=np.int64)
        if excl_zero.any():
            bad_ref = self.int_to_ref[excl_zero]
            bad_own = self.row_owner_int[excl_zero]
            o = np.lexsort((bad_ref, bad_own))
            bo, br = bad_own[o], bad_ref[o]
            firsts = np.r_[True, bo[1:] != bo[:-1]]
            first_bad[bo[firsts]] = br[firsts]
        self.sub_first_bad = first_bad.astype(np.int32)

        # columns
        col_owner = cm["col_owner"].astype(np.int64)
        self.col_owner = col_owner.astype(np.int32)
        self.col_len = sup_len[col_owner].astype(np.int32)
        self.col_rowbase = self.row_start[ball_idx[ball_ptr[:-1]]][col_owner].astype(np.int64)

        # reference slot -> internal slot per subsystem (its support
        # permutation). All subsystems at small N / exact mode / generic
        # graphs; at scale only one representative per structural id
        # (classes.sub_struct), the rest is materialised on demand.
        self._owner_ref, self._local_of_ref, self._mask = owner_ref, local_of_ref, mask
        self._sup_len = sup_len
        struct = classes.sub_struct if classes.sub_struct is not None else np.arange(n_sub)
        struct = np.asarray(struct, dtype=np.int64)
        full = n_sub <= 20000 or self.exact or not self.contiguous or classes.sub_struct is None
        self.ref_pos = self._ref_pos_rows(np.arange(n_sub)) if full else None
        if not self.contiguous:
            rptr, rows = mask._rows_of()
            j_of = np.repeat(np.arange(n_sub, dtype=np.int64), np.diff(rptr))
            slot = np.arange(rows.size) - np.repeat(rptr[:-1], np.diff(rptr))
            self.col_irow = np.zeros((n_sub, self.s_pad), dtype=np.int32)
            self.col_irow[j_of, self.ref_pos[j_of, slot]] = self.ref_to_int[rows]
        else:
            self.col_irow = None
        perm_keys, perm_of = {}, {}
        if full:
            perm_id = np.empty(n_sub, dtype=np.int64)
            for j in range(n_sub):
                key = self.ref_pos[j, :sup_len[j]].tobytes()
                if key not in perm_keys:
                    perm_keys[key] = len(perm_keys)
                    perm_of[perm_keys[key]] = self.ref_pos[j, :sup_len[j]].astype(np.int64)
                perm_id[j] = perm_keys[key]
        else:
            _, rep_sub, sinv = np.unique(struct, return_index=True, return_inverse=True)
            rows_rep = self._ref_pos_rows(rep_sub)
            sid = np.empty(rep_sub.size, dtype=np.int64)
            for u, r in enumerate(rep_sub.tolist()):
                pv = rows_rep[u, :sup_len[r]].astype(np.int64)
                key = pv.tobytes()
                if key not in perm_keys:
                    perm_keys[key] = len(perm_keys)
                    perm_of[perm_keys[key]] = pv
                sid[u] = perm_keys[key]
            perm_id = sid[sinv.ravel()]

        # device classes = (host class, support permutation)
        col_perm = perm_id[col_owner]
        pairs = np.stack([classes.col_class.astype(np.int64), col_perm], axis=1)
        upairs, dev_class = np.unique(pairs, axis=0, return_inverse=True)
        dev_class = dev_class.ravel()
        n_cls = upairs.shape[0]
        self.n_classes = n_cls
        self.col_class = dev_class.astype(np.int32)
        cls_s, cls_n0, cls_ldn, cls_m = [], [], [], []
        null_blocks, g_blocks, p_blocks = [], [], []
        self._class_perm = []
        for k in range(n_cls):
            hc = classes.classes[int(upairs[k, 0])]
            perm = perm_of[int(upairs[k, 1])]
            s = int(perm.size)
            self._class_perm.append(perm)
            null = hc.null
            n0 = null.shape[1]
            ldn = _ld_frag(_round(n0, 8))
            blk = np.zeros((_round(s, 8), ldn))
            blk[perm, :n0] = null
            null_blocks.append(blk.ravel())
            cls_s.append(s); cls_n0.append(n0); cls_ldn.append(ldn); cls_m.append(hc.g.shape[0])
            if self.exact:
                g_blocks.append(np.ascontiguousarray(hc.g).ravel())
                p_blocks.append(np.ascontiguousarray(hc.projector).ravel())
        self.class_s = np.array(cls_s, dtype=np.int32)
        self.class_n0 = np.array(cls_n0, dtype=np.int32)
        self.class_ldn = np.array(cls_ldn, dtype=np.int32)
        self.class_m = np.array(cls_m, dtype=np.int32)
        self.class_null_off = np.concatenate([[0], np.cumsum([b.size for b in null_blocks])]).astype(np.int64)
        self.null_pool = np.concatenate(null_blocks) if null_blocks else np.zeros(1)
        if self.exact:
            self.class_g_off = np.concatenate([[0], np.cumsum([b.size for b in g_blocks])]).astype(np.int64)
            self.class_p_off = np.concatenate([[0], np.cumsum([b.size for b in p_blocks])]).astype(np.int64)
            self.g_pool = np.concatenate(g_blocks)
            self.p_pool = np.concatenate(p_blocks)
        self.m_pad = _round(max(cls_m) if cls_m else 1, 4)

        # particular solution q (internal order) and reduced rhs, one per
        # distinct (device class, rhs)
        vpairs = np.stack([dev_class.astype(np.int64), classes.col_rhs], axis=1)
        uv, col_vec = np.unique(vpairs, axis=0, return_inverse=True)
        col_vec = col_vec.ravel()
        q_list, rhs_list = [], []
        for k, rid in uv.tolist():
            hc = classes.classes[int(upairs[k, 0])]
            rhs = classes.rhs_table[rid]
            q = np.zeros(self.s_pad)
            q[self._class_perm[k]] = hc.projector @ rhs
            r = np.zeros(self.m_pad)
            r[:rhs.size] = rhs
            q_list.append(q)
            rhs_list.append(r)
        self.col_vec = col_vec.astype(np.int32)

        # audit tables (on-device verify_fixed_point): per device class the
        # reference's touched-rows operator g0 (reference support order) and
        # the support permutation; per column the rhs0 pin
        if classes.col_pin is not None:
            g0s = [np.ascontiguousarray(classes.classes[int(upairs[k, 0])].g0) for k in range(n_cls)]
            self.class_ntouch = np.array([g.shape[0] for g in g0s], dtype=np.int32)
            self.class_g0_off = np.concatenate([[0], np.cumsum([g.size for g in g0s])]).astype(np.int64)
            self.g0_pool = np.concatenate([g.ravel() for g in g0s])
            self.class_perm_off = np.concatenate([[0], np.cumsum([p_.size for p_ in self._class_perm])]).astype(np.int64)
            self.perm_pool = np.concatenate(self._class_perm).astype(np.int32)
            self.col_pin = classes.col_pin.astype(np.int32)
        else:
            self.class_ntouch = self.class_g0_off = self.g0_pool = None
            self.class_perm_off = self.perm_pool = self.col_pin = None
        self.n_vec = len(q_list)
        self.q_pool = np.concatenate(q_list)
        self.rhs_pool = np.concatenate(rhs_list)

        # tiles of same-class columns
        self.tile_cols = int(tile_cols) if tile_cols else choose_tile_cols(n_x)
        owned = np.arange(*self.own_cols)
        order = owned[np.lexsort((owned, dev_class[owned]))]
        self.tile_colv = np.zeros(n_x, dtype=np.int32)
        self.tile_colv[:order.size] = order
        tcls, tfirst, tcount = [], [], []
        sorted_cls = dev_class[order]
        bounds = np.flatnonzero(np.r_[True, sorted_cls[1:] != sorted_cls[:-1], True])
        for a, b in zip(bounds[:-1], bounds[1:]):
            for f in range(a, b, self.tile_cols):
                tcls.append(int(sorted_cls[a])); tfirst.append(f); tcount.append(min(self.tile_cols, b - f))
        self.tile_class = np.array(tcls, dtype=np.int32)
        self.tile_first = np.array(tfirst, dtype=np.int32)
        self.tile_count = np.array(tcount, dtype=np.int32)
        self.n_tiles = len(tcls)

        # plant CSR (sorted, as scipy stores it); absent for solve-only sessions
        if system is not None:
            a = system.a.tocsr(); a.sort_indices()
            b = system.b.tocsr(); b.sort_indices()
        else:
            import scipy.sparse as _sp
            a, b = _sp.csr_matrix((n_x, n_x)), _sp.csr_matrix((n_x, max(n_u, 0)))
        self.has_plant = system is not None
        self.a_ptr, self.a_idx, self.a_val = a.indptr.astype(np.int64), a.indices.astype(np.int32), a.data.astype(np.float64)
        self.b_ptr, self.b_idx, self.b_val = b.indptr.astype(np.int64), b.indices.astype(np.int32), b.data.astype(np.float64)
        iown = np.repeat(np.arange(n_sub, dtype=np.int64), cm["input_count"])
        self.input_owner = iown.astype(np.int32)
        self.input_local = (self.ref_to_int[n_x * t + np.arange(n_u)] - self.row_start[iown]).astype(np.int32) \
            if n_u else np.zeros(0, np.int32)

    def _ref_pos_rows(self, subs):
        """Internal slot of every reference support slot, for the given
        subsystems (rows of a [len(subs), s_pad] int32 array)."""
        from .system_model import support_rows
        subs = np.asarray(subs, dtype=np.int64)
        ptr, rows = support_rows(self._mask, subs)
        lens = np.diff(ptr)
        k_of = np.repeat(np.arange(subs.size, dtype=np.int64), lens)
        j_of = subs[k_of]
        i_of = self._owner_ref[rows]
        e = np.searchsorted(self._key_e, i_of * self.n_sub + j_of)
        pos = self.ball_off[e].astype(np.int64) + self._local_of_ref[rows]
        slot = np.arange(rows.size) - np.repeat(ptr[:-1], lens)
        out = np.zeros((subs.size, self.s_pad), dtype=np.int32)
        out[k_of, slot] = pos
        return out

    def full_ref_pos(self):
        if self.ref_pos is None:
            self.ref_pos = self._ref_pos_rows(np.arange(self.n_sub))
        return self.ref_pos

    # -- maps to the reference layouts ------------------------------------------
    def column_gather(self, tables):
        """flat internal index of every reference column-layout cell (-1 at pads)."""
        cc, jj = np.nonzero(tables.col_valid)
        owner = self.col_owner[cc].astype(np.int64)
        out = np.full((tables.n_cols, tables.d_col), -1, dtype=np.int64)
        out[cc, jj] = cc * self.s_pad + self.full_ref_pos()[owner, jj]
        return out

    def row_gather(self, tables):
        """flat internal index of every reference row-layout cell (-1 at pads)."""
        rr, kk = np.nonzero(tables.row_valid)
        c = tables.rs[rr, kk]
        i = self.row_owner_int[self.ref_to_int[rr]].astype(np.int64)
        j = self.col_owner[c].astype(np.int64)
        e = np.searchsorted(self._key_e, i * self.n_sub + j)
        local = self.ref_to_int[rr] - self.row_start[i]
        out = np.full((tables.n_rows, tables.d_row), -1, dtype=np.int64)
        out[rr, kk] = c * self.s_pad + self.ball_off[e].astype(np.int64) + local
        return out

    def smem_estimate(self):
        s8 = _round(int(self.class_s.max()), 8)
        n08 = _round(int(self.class_n0.max()), 8)
        ldk = _ld_frag(self.tile_cols)
        return 8 * (s8 * int(self.class_ldn.max()) + s8 * ldk + 5 * n08 * ldk + 64)
