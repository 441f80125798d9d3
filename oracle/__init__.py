"""ORACLE — test infrastructure only.

A CPU restatement of the HSZ reference (arXiv 2603.25206, /root/reference/pkg)
used exclusively as the *checker*: by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg.  The product
package ``paper_2603_25206_b200`` never imports, links or executes anything in
this directory; its data path is the CUDA library ``libhszg.so`` and it fails
loudly when that library is missing.

Parity pinning: ``tests/golden/`` holds fixtures produced by importing the real
reference package in the build container (``tests/golden/make_golden.py``); the
CPU test-suite checks this oracle against them (``tests/test_oracle_golden.py``).
The N1–N5 operations (variance, regional statistics, threshold count, gradient
magnitude) have no reference implementation; their oracle definitions follow
SURVEY.md §8(a) and are built on the pinned stage-③ outputs.
"""
