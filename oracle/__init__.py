"""TEST INFRASTRUCTURE ONLY — CPU oracle for the l1 solver hot path.

Nothing in ``paper_1007_3753_b200`` may import this package.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm use it, and only as the checker or the timed CPU baseline.

Parity status: PINNED.  ``tests/golden/make_golden.py`` runs the real
reference package (``/root/reference/pkg``, compiled ``_accel``) in the
build container and commits its outputs as fixtures; ``tests/test_oracle_pins.py``
checks this restatement against those fixtures bit-for-bit (iteration counts,
trace) and to 1e-12 on the iterates.
"""

from oracle.l1_oracle import *  # noqa: F401,F403
