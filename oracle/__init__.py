"""CPU oracle for the manigraph (A, B) formation + LOBPCG path.

TEST INFRASTRUCTURE ONLY.  Nothing under ``paper_2112_07862_b200/`` imports
this package; only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may use it, and
only as the checker or as the timed CPU baseline -- never as the product.

The oracle is pinned against golden vectors produced by the unmodified
reference (``tests/golden/make_golden.py`` imports ``/root/reference/pkg/src``
in the build container and writes ``tests/golden/*.npz``); see
``tests/test_oracle_golden.py``.
"""

from .mg_oracle import *  # noqa: F401,F403
