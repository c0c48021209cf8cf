"""Plant, interconnection graph and d-hop locality structure (host-side setup).

Same public surface as `/root/reference/pkg/src/locality_mpc/system_model.py`
(`SubsystemPartition` 30-87, `SubsystemGraph` 90-135, `graph_distance`
138-159, `LtiSystem` 162-201, `build_chain_network` 204-240,
`phi_row_owners` 243-252, `LocalityMask` 255-280, `build_locality_mask`
283-330, `longest_vector_lengths` 333-337, `lemma1_bounds` 340-361), built
for network sizes the reference cannot reach: every structure is produced by
array operations instead of per-node Python loops, and the mask keeps a
compact per-subsystem description (balls + ownership) from which the
per-row/per-column support tuples of the reference are materialised only on
first access. The device layout (`devlayout.py`) is built from the compact
form directly.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

UNREACHABLE = math.inf

# Chain benchmark blocks (reference system_model.py:26-27).
CHAIN_A_DIAG = np.array([[1.0, 0.1], [-0.3, 0.7]])
CHAIN_A_COUPLING = np.array([[0.0, 0.0], [0.1, 0.1]])


def _ranges_to_owner(ranges, total):
    bounds = np.array([b for _, b in ranges], dtype=np.int64)
    # index k belongs to the first range whose stop exceeds k
    return np.searchsorted(bounds, np.arange(total, dtype=np.int64), side="right").astype(np.int32)


@dataclass(frozen=True)
class SubsystemPartition:
    """Contiguous half-open state/input ranges, one pair per subsystem."""

    state_ranges: tuple
    input_ranges: tuple

    def __post_init__(self):
        if len(self.state_ranges) != len(self.input_ranges):
            raise ValueError("state and input range lists must have equal length")
        if len(self.state_ranges) == 0:
            raise ValueError("partition needs at least one subsystem")
        st = np.asarray(self.state_ranges, dtype=np.int64).reshape(-1, 2)
        ip = np.asarray(self.input_ranges, dtype=np.int64).reshape(-1, 2)
        starts = np.concatenate([[0], st[:-1, 1]])
        bad = np.nonzero((st[:, 0] != starts) | (st[:, 1] <= st[:, 0]))[0]
        if bad.size:
            raise ValueError(f"state ranges must tile [0, n_states); bad range {int(bad[0])}")
        starts = np.concatenate([[0], ip[:-1, 1]])
        bad = np.nonzero((ip[:, 0] != starts) | (ip[:, 1] < ip[:, 0]))[0]
        if bad.size:
            raise ValueError(f"input ranges must tile [0, n_inputs); bad range {int(bad[0])}")

    @property
    def subsystem_count(self) -> int:
        return len(self.state_ranges)

    @property
    def n_states(self) -> int:
        return int(self.state_ranges[-1][1])

    @property
    def n_inputs(self) -> int:
        return int(self.input_ranges[-1][1])

    def state_counts(self) -> np.ndarray:
        st = np.asarray(self.state_ranges, dtype=np.int64).reshape(-1, 2)
        return st[:, 1] - st[:, 0]

    def input_counts(self) -> np.ndarray:
        ip = np.asarray(self.input_ranges, dtype=np.int64).reshape(-1, 2)
        return ip[:, 1] - ip[:, 0]

    def state_owner(self) -> np.ndarray:
        return _ranges_to_owner(self.state_ranges, self.n_states)

    def input_owner(self) -> np.ndarray:
        return _ranges_to_owner(self.input_ranges, self.n_inputs)

    @classmethod
    def uniform(cls, n_subsystems: int, states_per: int, inputs_per: int) -> "SubsystemPartition":
        k = np.arange(n_subsystems + 1)
        s = tuple(zip((k[:-1] * states_per).tolist(), (k[1:] * states_per).tolist()))
        u = tuple(zip((k[:-1] * inputs_per).tolist(), (k[1:] * inputs_per).tolist()))
        return cls(s, u)


@dataclass(frozen=True)
class SubsystemGraph:
    """Undirected unweighted graph; `adjacency[i]` is a sorted int32 array."""

    node_count: int
    adjacency: tuple

    def __post_init__(self):
        if len(self.adjacency) != self.node_count:
            raise ValueError("adjacency list length must equal node_count")
        src, dst = self._edge_arrays()
        if np.any(src == dst):
            i = int(src[np.nonzero(src == dst)[0][0]])
            raise ValueError(f"self-loop at node {i}")
        out = (dst < 0) | (dst >= self.node_count)
        if np.any(out):
            k = int(np.nonzero(out)[0][0])
            raise ValueError(f"neighbor {int(dst[k])} of node {int(src[k])} out of range")
        fwd = src.astype(np.int64) * self.node_count + dst
        rev = dst.astype(np.int64) * self.node_count + src
        missing = ~np.isin(rev, fwd)
        if np.any(missing):
            k = int(np.nonzero(missing)[0][0])
            raise ValueError(f"edge ({int(src[k])},{int(dst[k])}) is not symmetric")

    def _edge_arrays(self):
        lens = np.fromiter((len(a) for a in self.adjacency), dtype=np.int64,
                           count=self.node_count)
        src = np.repeat(np.arange(self.node_count, dtype=np.int64), lens)
        dst = (np.concatenate([np.asarray(a, dtype=np.int64) for a in self.adjacency])
               if lens.sum() else np.zeros(0, dtype=np.int64))
        return src, dst

    @classmethod
    def from_edges(cls, node_count: int, edges) -> "SubsystemGraph":
        e = np.asarray(list(edges), dtype=np.int64).reshape(-1, 2)
        e = e[e[:, 0] != e[:, 1]]
        both = np.concatenate([e, e[:, ::-1]])
        key = np.unique(both[:, 0] * max(node_count, 1) + both[:, 1])
        src, dst = key // max(node_count, 1), key % max(node_count, 1)
        split = np.searchsorted(src, np.arange(node_count + 1))
        adj = tuple(dst[split[i]:split[i + 1]].astype(np.int32) for i in range(node_count))
        return cls(node_count, adj)

    @property
    def max_degree(self) -> int:
        return max((len(a) for a in self.adjacency), default=0)

    def adjacency_matrix(self) -> sp.csr_matrix:
        src, dst = self._edge_arrays()
        n = self.node_count
        return sp.csr_matrix((np.ones(src.size, dtype=np.int8), (src, dst)), shape=(n, n))

    def ball(self, node: int, radius: int) -> np.ndarray:
        """Sorted node ids within `radius` hops of `node` (closed ball)."""
        seen = np.zeros(self.node_count, dtype=bool)
        seen[node] = True
        frontier = np.array([node], dtype=np.int64)
        for _ in range(radius):
            if frontier.size == 0:
                break
            nxt = np.concatenate([np.asarray(self.adjacency[v], dtype=np.int64)
                                  for v in frontier])
            nxt = np.unique(nxt[~seen[nxt]])
            seen[nxt] = True
            frontier = nxt
        return np.nonzero(seen)[0].astype(np.int32)

    def balls(self, radius: int):
        """All closed balls at once, as CSR (indptr, sorted indices)."""
        n = self.node_count
        step = self.adjacency_matrix() + sp.identity(n, dtype=np.int8, format="csr")
        step.data[:] = 1
        reach = sp.identity(n, dtype=np.int8, format="csr")
        for _ in range(radius):
            nxt = (reach @ step).tocsr()
            nxt.data[:] = 1
            if nxt.nnz == reach.nnz:
                break
            reach = nxt
        reach.sort_indices()
        return reach.indptr.astype(np.int64), reach.indices.astype(np.int32)


def graph_distance(graph: SubsystemGraph, i: int, j: int):
    """Hop count between i and j; 0 for i == j, `UNREACHABLE` across components."""
    n = graph.node_count
    if not (0 <= i < n and 0 <= j < n):
        raise ValueError(f"node ids ({i}, {j}) out of range for {n} nodes")
    if i == j:
        return 0
    seen = np.zeros(n, dtype=bool)
    seen[i] = True
    frontier = np.array([i], dtype=np.int64)
    hops = 0
    while frontier.size:
        hops += 1
        nxt = np.concatenate([np.asarray(graph.adjacency[v], dtype=np.int64) for v in frontier])
        nxt = np.unique(nxt[~seen[nxt]])
        if np.any(nxt == j):
            return hops
        seen[nxt] = True
        frontier = nxt
    return UNREACHABLE


@dataclass(frozen=True)
class LtiSystem:
    """x+ = A x + B u with block sparsity following the subsystem graph."""

    a: sp.csr_matrix
    b: sp.csr_matrix
    partition: SubsystemPartition
    graph: SubsystemGraph

    def __post_init__(self):
        p = self.partition
        if self.a.shape != (p.n_states, p.n_states):
            raise ValueError("A shape inconsistent with partition")
        if self.b.shape != (p.n_states, p.n_inputs):
            raise ValueError("B shape inconsistent with partition")
        if self.graph.node_count != p.subsystem_count:
            raise ValueError("graph node count must match subsystem count")
        adj = self.graph.adjacency_matrix().tocsr()
        sown, iown = p.state_owner(), p.input_owner()
        for name, mat, col_owner in (("A", self.a, sown), ("B", self.b, iown)):
            coo = mat.tocoo()
            r, c = sown[coo.row], col_owner[coo.col]
            off = r != c
            if np.any(off):
                linked = np.asarray(adj[r[off], c[off]]).ravel() != 0
                if not np.all(linked):
                    k = int(np.nonzero(~linked)[0][0])
                    raise ValueError(f"{name} couples subsystems ({int(r[off][k])},"
                                     f"{int(c[off][k])}) outside the graph")

    @property
    def n_states(self) -> int:
        return self.partition.n_states

    @property
    def n_inputs(self) -> int:
        return self.partition.n_inputs


def build_chain_network(n_subsystems: int, coupling_radius: int = 1,
                        two_inputs: bool = False) -> LtiSystem:
    """The two-state chain benchmark plant (reference system_model.py:204-240)."""
    n = int(n_subsystems)
    if n < 1:
        raise ValueError("need at least one subsystem")
    if coupling_radius < 1:
        raise ValueError("coupling_radius must be >= 1")
    nu_per = 2 if two_inputs else 1
    part = SubsystemPartition.uniform(n, 2, nu_per)
    i = np.arange(n)
    offs = [o for o in range(-coupling_radius, coupling_radius + 1) if o != 0]
    inside = [(i + o >= 0) & (i + o < n) for o in offs]
    pairs_i = np.concatenate([i] + [i[m] for m in inside])
    pairs_j = np.concatenate([i] + [i[m] + o for m, o in zip(inside, offs)])
    blocks = np.concatenate([np.broadcast_to(CHAIN_A_DIAG, (n, 2, 2))] +
                            [np.broadcast_to(CHAIN_A_COUPLING, (int(m.sum()), 2, 2))
                             for m in inside])
    rr = (2 * pairs_i)[:, None, None] + np.arange(2)[None, :, None]
    cc = (2 * pairs_j)[:, None, None] + np.arange(2)[None, None, :]
    rr, cc = np.broadcast_arrays(rr, cc)
    vals = blocks.reshape(-1)
    keep = vals != 0.0
    a = sp.coo_matrix((vals[keep], (rr.reshape(-1)[keep], cc.reshape(-1)[keep])),
                      shape=(2 * n, 2 * n)).tocsr()
    if two_inputs:
        b = sp.identity(2 * n, format="csr", dtype=np.float64)
    else:
        b = sp.csr_matrix((np.ones(2 * n), (np.arange(2 * n), np.repeat(i, 2))), shape=(2 * n, n))
    a.sort_indices()
    b.sort_indices()
    edges = np.stack([pairs_i[n:], pairs_j[n:]], axis=1)
    graph = SubsystemGraph.from_edges(n, edges[edges[:, 0] < edges[:, 1]])
    return LtiSystem(a, b, part, graph)


def phi_row_owners(partition: SubsystemPartition, horizon: int) -> np.ndarray:
    """Owner subsystem of each stacked response row (states time-major, then inputs)."""
    return np.concatenate([np.tile(partition.state_owner(), horizon),
                           np.tile(partition.input_owner(), horizon - 1)])


class LocalityMask:
    """Support of the stacked response under the d-hop rule.

    Public fields follow the reference (`system_model.py:255-280`):
    `n_rows, n_cols, d, row_supports, col_supports, d_row, d_col, n_entries`.
    When built by `build_locality_mask` the mask also carries its compact
    form -- closed balls as CSR (`ball_ptr`, `ball_idx`), the partition and
    the horizon -- and materialises the per-row / per-column tuples lazily,
    so an N=10^6 mask costs O(N) memory until someone asks for them.
    """

    def __init__(self, n_rows, n_cols, d, row_supports=None, col_supports=None, *,
                 compact=None):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.d = int(d)
        self._row_supports = None if row_supports is None else tuple(row_supports)
        self._col_supports = None if col_supports is None else tuple(col_supports)
        self.compact = compact
        if compact is not None:
            self.d_row = int(compact["row_len_sub"].max())
            self.d_col = int(compact["col_len_sub"].max())
            self._n_entries = int((compact["row_len_sub"] * compact["rows_per_sub"]).sum())
        else:
            if self._row_supports is None or self._col_supports is None:
                raise ValueError("explicit masks need both support tuples")
            self.d_row = max(len(s) for s in self._row_supports)
            self.d_col = max(len(s) for s in self._col_supports)
            self._n_entries = sum(len(s) for s in self._row_supports)

    # --- compact-form helpers -------------------------------------------------
    def _cols_of(self):
        c = self.compact
        if "cols_of" not in c:
            c["cols_of"] = _expand_ball_ranges(c["ball_ptr"], c["ball_idx"],
                                               c["state_start"], c["state_count"])
        return c["cols_of"]

    def _rows_of(self):
        c = self.compact
        if "rows_of" not in c:
            c["rows_of"] = _ball_row_sets(c)
        return c["rows_of"]

    @property
    def row_supports(self):
        if self._row_supports is None:
            ptr, idx = self._cols_of()
            per_sub = [idx[ptr[i]:ptr[i + 1]] for i in range(len(ptr) - 1)]
            owners = self.compact["row_owner"]
            self._row_supports = tuple(per_sub[o] for o in owners.tolist())
        return self._row_supports

    @property
    def col_supports(self):
        if self._col_supports is None:
            ptr, idx = self._rows_of()
            per_sub = [idx[ptr[i]:ptr[i + 1]] for i in range(len(ptr) - 1)]
            owners = self.compact["col_owner"]
            self._col_supports = tuple(per_sub[o] for o in owners.tolist())
        return self._col_supports

    @property
    def n_entries(self) -> int:
        return self._n_entries


def _expand_ball_ranges(ball_ptr, ball_idx, start, count):
    """For each node, concatenate the index ranges [start[j], start[j]+count[j])
    of its ball members j, in ball order. Returns CSR (ptr, idx)."""
    lens = count[ball_idx]
    per_node = np.add.reduceat(lens, ball_ptr[:-1]) if ball_idx.size else np.zeros(0, np.int64)
    per_node = np.where(np.diff(ball_ptr) > 0, per_node, 0)
    ptr = np.concatenate([[0], np.cumsum(per_node)]).astype(np.int64)
    seg_start = np.repeat(start[ball_idx], lens)
    seg_off = np.arange(lens.sum(), dtype=np.int64) - np.repeat(np.cumsum(lens) - lens, lens)
    return ptr, (seg_start + seg_off).astype(np.int64)


def _ball_row_sets(c):
    """Column supports per subsystem: for each time block (states, then
    inputs) the signal rows of every ball member, time-major
    (reference system_model.py:310-324)."""
    n_x, n_u, t = c["n_x"], c["n_u"], c["horizon"]
    ball_ptr, ball_idx = c["ball_ptr"], c["ball_idx"]
    parts_ptr = []
    parts_idx = []
    for tt in range(t):
        parts = _expand_ball_ranges(ball_ptr, ball_idx, c["state_start"] + tt * n_x, c["state_count"])
        parts_ptr.append(parts[0]); parts_idx.append(parts[1])
    for tt in range(t - 1):
        parts = _expand_ball_ranges(ball_ptr, ball_idx, c["input_start"] + n_x * t + tt * n_u,
                                    c["input_count"])
        parts_ptr.append(parts[0]); parts_idx.append(parts[1])
    n = len(ball_ptr) - 1
    lens = np.stack([np.diff(p) for p in parts_ptr], axis=1)       # (n, blocks)
    total = lens.sum(axis=1)
    ptr = np.concatenate([[0], np.cumsum(total)]).astype(np.int64)
    out = np.empty(int(ptr[-1]), dtype=np.int64)
    # destination offset of block b for node i = ptr[i] + sum(lens[i, :b])
    blk_off = ptr[:-1, None] + np.cumsum(lens, axis=1) - lens
    for b, (pp, ii) in enumerate(zip(parts_ptr, parts_idx)):
        l = np.diff(pp)
        dst = np.repeat(blk_off[:, b], l) + (np.arange(l.sum()) - np.repeat(pp[:-1], l))
        out[dst] = ii
    return ptr, out


def support_rows(mask: LocalityMask, subs):
    """Column supports (reference row indices, reference order) of the given
    subsystems only, as CSR (ptr, rows) -- without materialising all of them."""
    c = mask.compact
    subs = np.asarray(subs, dtype=np.int64)
    bp, bi = c["ball_ptr"], c["ball_idx"]
    lens = bp[subs + 1] - bp[subs]
    ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    idx = bi[np.repeat(bp[subs], lens) + (np.arange(lens.sum()) - np.repeat(ptr[:-1], lens))]
    sub = dict(c)
    sub["ball_ptr"], sub["ball_idx"] = ptr, idx
    return _ball_row_sets(sub)


def build_locality_mask(system: LtiSystem, d: int, horizon: int) -> LocalityMask:
    """d-hop closed-ball mask over the horizon (reference system_model.py:283-330)."""
    if horizon < 2:
        raise ValueError("horizon must be >= 2")
    if d < 0:
        raise ValueError("hop radius must be >= 0")
    part, graph = system.partition, system.graph
    t = int(horizon)
    n_x, n_u = part.n_states, part.n_inputs
    ball_ptr, ball_idx = graph.balls(d)
    st = np.asarray(part.state_ranges, dtype=np.int64).reshape(-1, 2)
    ip = np.asarray(part.input_ranges, dtype=np.int64).reshape(-1, 2)
    s_cnt, u_cnt = st[:, 1] - st[:, 0], ip[:, 1] - ip[:, 0]
    ball_sx = np.add.reduceat(s_cnt[ball_idx], ball_ptr[:-1])
    ball_su = np.add.reduceat(u_cnt[ball_idx], ball_ptr[:-1])
    compact = {
        "ball_ptr": ball_ptr, "ball_idx": ball_idx,
        "state_start": st[:, 0], "state_count": s_cnt,
        "input_start": ip[:, 0], "input_count": u_cnt,
        "n_x": n_x, "n_u": n_u, "horizon": t,
        "row_owner": phi_row_owners(part, t).astype(np.int64),
        "col_owner": part.state_owner().astype(np.int64),
        # support length of each subsystem's rows / columns
        "row_len_sub": ball_sx.astype(np.int64),
        "col_len_sub": (t * ball_sx + (t - 1) * ball_su).astype(np.int64),
        # rows owned per subsystem (states x T + inputs x (T-1))
        "rows_per_sub": (t * s_cnt + (t - 1) * u_cnt).astype(np.int64),
    }
    return LocalityMask(n_x * t + n_u * (t - 1), n_x, d, compact=compact)


def longest_vector_lengths(mask: LocalityMask):
    """(d_row, d_col): the padded strides of the two layouts."""
    return mask.d_row, mask.d_col


def lemma1_bounds(s: int, l: int, d: int, horizon: int):
    """Lemma 1 bounds on (d_row, d_col) (reference system_model.py:340-361)."""
    if s < 1 or horizon < 2 or d < 0 or l < 0:
        raise ValueError("need s >= 1, horizon >= 2, d >= 0, l >= 0")
    if l <= 1:
        nodes = 1 if l == 0 else d + 1
    else:
        nodes = (l ** (d + 1) - 1) // (l - 1)
    row = s * nodes
    return row, (2 * horizon - 1) * row
