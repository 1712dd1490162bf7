"""ORACLE — test infrastructure only.

A CPU restatement of the reference KVServe codec pipeline
(``/root/reference/pkg/src/kvpilot/pipeline``) used exclusively as the
*checker* for the CUDA path: by ``tests/``, ``__graft_entry__.smoke()`` and
the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``.  The
product package ``paper_2605_13734_b200`` never imports this package, and
its GPU path fails loudly when its CUDA library is missing instead of
falling back here.

Pinning: ``tests/test_oracle_pins.py`` checks this restatement against the
reference itself (imported from /root/reference when present) and against
the committed golden fixtures in ``tests/golden/`` that
``tests/golden/make_golden.py`` generated from the unmodified reference.
The extension features the reference lacks (per-channel groups, affine
transform, per-layer / per-token mixed precision, block framing) are
restated in ``oracle.extensions`` on top of the pinned primitives; their
*layout conventions* are parity-unpinned.
"""

from oracle.pipeline import *  # noqa: F401,F403
from oracle.pipeline import __all__ as _p_all
from oracle.extensions import *  # noqa: F401,F403
from oracle.extensions import __all__ as _e_all

__all__ = list(_p_all) + list(_e_all)
