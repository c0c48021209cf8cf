"""The persistent kernels under the bounds-checked build.

compute-sanitizer is closed on the GPU pool (profiles/sanitize_r02.txt), so
the library is also built with -DDLMPC_CHECKED (libdlmpc_checked.so): every
epilogue store must hit an OWNED support cell of the column layout, every Φ
load a cell of the layout, every Φ-partial store its buffer, every TMA bulk
copy a source range inside ψ / λ and a destination inside the CTA's shared
memory plan. The first violation is recorded on the device and fails the
call (DeviceError). These runs cover the patch (GEMV pair), stream (TMA,
mbarriers, warp split), two-phase and exact kernels and the reference-layout
schedules; they also check run-to-run determinism, the observable symptom of
a data race.
"""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2103_14990_b200", "libdlmpc_checked.so")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def checked_lib():
    import build
    return build.build(checked=True)


def test_checked_build_kernels_stay_in_bounds(checked_lib):
    env = dict(os.environ, DLMPC_LIB=checked_lib)
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py")], env=env,
                         capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "== case sched" in res.stdout


def test_checked_build_parity_subset(checked_lib):
    """A slice of the parity suite itself on the checked library: the golden
    closed loops (patch kernels, both arithmetic flavours), the stream kernel
    against the patch kernel, and the partitioned ranks (owned-range stores)."""
    env = dict(os.environ, DLMPC_LIB=checked_lib)
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                          os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                          os.path.join(ROOT, "tests", "test_gpu_partitioned.py"),
                          "-k", "closed_loops_against_reference or stream_and_patch or partitioned_closed_loop "
                                "or generic_graph or grid_network"],
                         env=env, capture_output=True, text=True, timeout=1800, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]


@pytest.mark.parametrize("case", ["c2", "stream", "twophase"])
def test_run_to_run_bitwise(case, monkeypatch):
    """Ten repeats of a closed loop give bit-identical trajectories (races in
    the grid barrier, the TMA / mbarrier pipeline or the Φ partial slots
    would show up as nondeterminism)."""
    import numpy as np
    import paper_2103_14990_b200 as pb
    n, env = {"c2": (100, {}), "stream": (2500, {"DLMPC_FORCE_STREAM": "1"}),
              "twophase": (300, {"DLMPC_FORCE_TWOPHASE": "1"})}[case]
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    system, spec, mask, x0 = pb.scenario_problem(pb.Scenario(n=n, d=3, horizon=10, seed=9))
    sess = pb.DlmpcSession(system, spec, mask, "b200")
    ref, _ = sess.simulate(x0, 3)
    for _ in range(9):
        t, _ = sess.simulate(x0, 3)
        assert t.step_iterations == ref.step_iterations
        assert np.array_equal(t.states, ref.states) and np.array_equal(t.inputs, ref.inputs)
    sess.close()
