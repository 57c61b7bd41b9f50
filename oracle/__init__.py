"""TEST INFRASTRUCTURE ONLY -- the CPU oracle of the SAME Gibbs path.

A NumPy restatement of the reference's algorithm (samegibbs 0.1.0,
/root/reference/pkg/src/samegibbs), used as the checker by ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py``.  The product package never imports it.

Parity pinning: every function is checked against golden vectors produced by
running the reference itself (``tests/golden/make_golden.py``, committed
fixtures ``tests/golden/*.npz``); see ``tests/test_oracle_golden.py``.
"""

from .samegibbs_oracle import *  # noqa: F401,F403
