"""CPU oracle for the DLMPC ADMM hot path -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` leg may import this package, and only as the checker or
as the timed CPU baseline. The product (`paper_2103_14990_b200`) never
imports it and has no CPU fallback.

`admm_ref.py` restates the reference's per-iteration arithmetic
(`/root/reference/pkg/src/locality_mpc/admm.py:155-217, 315-369`,
`sls_core.py:37-47, 330-349, 442-472`) in numpy with the same operation
order (numpy pairwise `.sum(axis=-1)` for the Ψ reductions, strict
left-to-right dots elsewhere, no FMA), so its iterates are bit-identical to
the reference's `sequential` schedule. Parity is pinned against golden
vectors produced by running the reference itself
(`tests/golden/make_golden.py` -> `tests/golden/*.npz`) and against the
known answers of SURVEY.md Appendix B.
"""
