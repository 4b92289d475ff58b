"""B200-native Random SubMatrix (RSM, arXiv 1411.0814) hot path.

Host API: :mod:`paper_1411_0814_b200.rsm` (mirror of the reference ``rsm::``
C++ API) over the C-ABI in ``include/rsm_b200.h``, implemented by the sm_100a
library ``librsm_b200.so`` built from ``csrc/``.
"""
from . import rsm  # noqa: F401
