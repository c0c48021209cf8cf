import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)

GOLDEN = os.path.join(TESTS, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def golden(name):
    path = os.path.join(GOLDEN, name + ".npz")
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


def chain_bundle(n, horizon, d, bounded=True, eps=1e-4, max_iters=5000, coupling_radius=1,
                 two_inputs=False):
    """Setup objects for the chain benchmark (mirrors the reference's
    tests/conftest.py:13-25 build_bundle)."""
    import paper_2103_14990_b200 as pb
    system = pb.build_chain_network(n, coupling_radius, two_inputs)
    spec = pb.make_benchmark_spec(system, horizon, eps=eps, bounded=bounded, max_iters=max_iters)
    mask = pb.build_locality_mask(system, d, horizon)
    tables = pb.LayoutTables(mask)
    op = pb.build_dynamics_operator(system, horizon)
    classes = pb.build_column_classes(op, mask)
    col_solvers = pb.precompute_column_solvers(op, mask, classes)
    return {"system": system, "spec": spec, "mask": mask, "tables": tables, "operator": op,
            "classes": classes, "col_solvers": col_solvers}


def random_graph_system(n, rng, p_edge=0.35, states_per=2):
    """A plant on a random connected graph with random blocks (non-contiguous
    balls: exercises the generic col_irow path)."""
    import scipy.sparse as sp
    import paper_2103_14990_b200 as pb
    edges = [(i, i + 1) for i in range(n - 1)]
    edges += [(i, j) for i in range(n) for j in range(i + 2, n) if rng.random() < p_edge]
    graph = pb.SubsystemGraph.from_edges(n, edges)
    part = pb.SubsystemPartition.uniform(n, states_per, 1)
    a = sp.lil_matrix((states_per * n, states_per * n))
    b = sp.lil_matrix((states_per * n, n))
    for i in range(n):
        s = slice(states_per * i, states_per * (i + 1))
        a[s, s] = rng.uniform(-0.5, 0.5, (states_per, states_per))
        b[s, i] = rng.uniform(0.5, 1.0, (states_per, 1))
        for j in graph.adjacency[i]:
            a[s, states_per * j:states_per * (j + 1)] = rng.uniform(-0.2, 0.2, (states_per, states_per))
    return pb.LtiSystem(a.tocsr(), b.tocsr(), part, graph)


def grid_network(rows, cols):
    """A 2-D grid of the chain's subsystems (2 states, 1 input; the chain's
    self and coupling blocks, coupled to the 4 grid neighbours), built through
    the generic LtiSystem / SubsystemGraph.from_edges path (SURVEY §8(d) C5:
    'a grid ... through the generic path'). Balls are diamonds, not
    contiguous id ranges: the two-phase kernel and the col_irow tables."""
    import scipy.sparse as sp
    import paper_2103_14990_b200 as pb
    n = rows * cols
    idx = lambda r, c: r * cols + c
    edges = [(idx(r, c), idx(r, c + 1)) for r in range(rows) for c in range(cols - 1)]
    edges += [(idx(r, c), idx(r + 1, c)) for r in range(rows - 1) for c in range(cols)]
    graph = pb.SubsystemGraph.from_edges(n, edges)
    part = pb.SubsystemPartition.uniform(n, 2, 1)
    a = sp.lil_matrix((2 * n, 2 * n))
    b = sp.lil_matrix((2 * n, n))
    for i in range(n):
        a[2 * i:2 * i + 2, 2 * i:2 * i + 2] = [[1.0, 0.1], [-0.3, 0.7]]
        b[2 * i, i] = 1.0
        b[2 * i + 1, i] = 1.0
        for j in graph.adjacency[i]:
            a[2 * i + 1, 2 * j:2 * j + 2] = [0.05, 0.05]
    return pb.LtiSystem(a.tocsr(), b.tocsr(), part, graph)
