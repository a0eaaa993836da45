"""CPU oracle for the CoR-UTV / ALM-CoRUTV hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (``cpu_baseline`` / ``--impl reference``) may import this package, and
only as the checker / the timed reference arm.  The product package
``paper_1906_04572_b200`` never imports it: the device path fails loudly when
its CUDA library is missing instead of falling back here.

Parity is pinned: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by the reference package itself
(``tests/golden/make_golden.py``, run in the build container where
``/root/reference`` is importable) and against the reference's own
known-answer tests (``pkg/tests/test_dense.py:97-115`` etc.).
"""

from .corutv_oracle import *  # noqa: F401,F403
from .corutv_oracle import __all__  # noqa: F401
