"""TEST SHIM -- lets the reference's own test-suite (pkg/tests, copied to
baseline/_ref_tests by tools/run_reference_tests.py) import `locality_mpc`
and run against paper_2103_14990_b200 unchanged.

Every name the tests use resolves to this package's device paths; the
reference's five schedule names are real device schedules. Three pieces the
package deliberately does not ship (SURVEY §2 OUT OF SCOPE) are supplied here
for the tests only:
  * the dense KKT oracle (`kkt_oracle_equality`, `simulate_with_oracle`) from
    oracle/kkt.py, the repo's pinned restatement of reference oracle.py;
  * `WorkerPool`, the reference's CPU thread pool: a stand-in so
    test_strategies.py imports (its TestWorkerPool cases are excluded);
  * `locality_mpc.bench` exposes the scenario API (Scenario, run_scenario,
    make_benchmark_spec, sample_initial_state); the sweep / CSV / SVG harness
    functions are absent (test_bench.py and the breakdown test are excluded).
"""

import sys
import types

import paper_2103_14990_b200 as _pb
from paper_2103_14990_b200 import *  # noqa: F401,F403
from paper_2103_14990_b200 import (admm, errors, report, scenario, sls_core, strategies,  # noqa: F401
                                   system_model)
from paper_2103_14990_b200.admm import Trajectory as _Trajectory

_strategies = types.ModuleType(__name__ + ".strategies")
_strategies.__dict__.update({k: v for k, v in strategies.__dict__.items() if not k.startswith("__")})


class WorkerPool:   # the reference's CPU pool is out of scope; import-only stand-in
    def __init__(self, worker_count):
        raise NotImplementedError("the CPU worker pool is replaced by the CUDA grid")


_strategies.WorkerPool = WorkerPool
_bench = types.ModuleType(__name__ + ".bench")
_bench.__dict__.update({k: v for k, v in scenario.__dict__.items() if not k.startswith("__")})

for _name, _mod in (("admm", admm), ("errors", errors), ("report", report), ("sls_core", sls_core),
                    ("strategies", _strategies), ("system_model", system_model), ("bench", _bench)):
    sys.modules[__name__ + "." + _name] = _mod
    globals()[_name] = _mod
WorkerPool = WorkerPool


def kkt_oracle_equality(spec, system, mask, x):
    from oracle.kkt import kkt_response
    return kkt_response(system, spec, mask, x)


def simulate_with_oracle(system, spec, mask, x0, t_sim):
    from oracle.kkt import kkt_closed_loop
    states, inputs = kkt_closed_loop(system, spec, mask, x0, t_sim)
    return _Trajectory(states, inputs, [])


__version__ = _pb.__version__
