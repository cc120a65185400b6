"""CPU oracle for the CSC Chebyshev-filter hot path — TEST INFRASTRUCTURE ONLY.

Nothing in the product package (``paper_1706_03591_b200``) imports this
package. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may use it, and only as the
checker or the timed CPU baseline, never as the thing measured or shipped.

Contents
--------
``csc_oracle``   numpy/scipy restatement of the reference's hot-path functions
                 (``pkg/src/cscluster/{filters,kmeans,graphs,signals,csc,dynamic}.py``),
                 each function citing the reference file:line it follows.
``cheb_filter.c`` plain-C restatement of ``apply_filter`` (filters.py:155-187,
                 with SciPy's ``csr_matvecs`` row loop inlined) and
                 ``_count_from_block`` (filters.py:190-196); OpenMP over rows
                 (per-row accumulation order is unchanged, so the result does
                 not depend on the thread count). Built by ``oracle/Makefile``
                 into ``oracle/build/liboracle.so``.
``native``       ctypes loader for that library.

Parity pin: the restatement is checked against golden vectors produced by the
live reference (``tests/golden/make_golden.py`` imports ``/root/reference``
in the build container and commits ``tests/golden/*.npz``); see
``tests/test_oracle_golden.py``.
"""
