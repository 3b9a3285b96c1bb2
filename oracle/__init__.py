"""TEST INFRASTRUCTURE ONLY — CPU oracle for the paulib_b200 hot path.

This package restates, on the CPU, the reference algorithm of
arxiv/paper_2605_25974's ``paulialg`` package (pure Python + numpy,
/root/reference/pkg/src/paulialg) for every function on the hot path, each
citing the reference file:line it follows.  It is the CHECKER: only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs
(``cpu_baseline`` and ``--impl reference``) may import it.  The product package
``paper_2605_25974_b200`` never imports it and has no CPU fallback.

Pinning: the restatement is checked against golden vectors produced by
running the reference itself (``tests/golden/make_golden.py`` imports
/root/reference/pkg/src/paulialg in the build container and commits the
outputs as ``tests/golden/*.npz``), plus the SPEC/PAPER known answers.
The reference's arithmetic lives in numpy (third party, un-vendored; pinned
by the reference only as ``numpy>=1.24``, pyproject.toml:10, effectively
>= 2.0 for ``np.bitwise_count``; numpy 2.3.5 here).

Modules:
  numpy_ref  numpy restatement (phase, sip, batched multiply, outer product,
             combine, greedy grouping, bitmatrix rows)
  cgreedy    ctypes wrapper of greedy.c, a plain-C restatement of the
             first-fit scan for full-size (config 3) parity runs
"""
