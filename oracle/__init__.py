"""CPU oracle for the ALISE hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import anything here,
and only as the checker or the timed CPU baseline.  The product package
``paper_2410_23537_b200`` never imports this package.

Parity pinning: the restatements here are checked against golden vectors
produced by the reference ``servesim`` package itself
(``tests/golden/make_golden.py``) and against the reference's own
known-answer tests (``pkg/tests/test_kvmanager.py``,
``pkg/tests/test_predictor.py``).
"""
