"""CPU oracle for the MBIR hot path -- TEST INFRASTRUCTURE ONLY.

A float64 numpy restatement of the reference algorithms (tomoforge, pure
numpy).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / ``--impl reference`` legs may import it, and only
as the checker or the timed CPU baseline.  The product package
``paper_2603_28756_b200`` never imports this module.

Parity pinning: ``tests/golden/make_golden.py`` ran the reference itself (from
/root/reference, importable in the build container) and committed its outputs
as ``tests/golden/*.npz``; ``tests/test_oracle.py`` checks this oracle against
every fixture, so the oracle is pinned to the reference, not to itself.
"""

from .tomoforge_oracle import *  # noqa: F401,F403
