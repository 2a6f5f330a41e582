"""B200-native Block-CUR hot path (arXiv 1703.06065) behind the reference's bcur:: API.

Import ``paper_1703_06065_b200.bcur`` for the reference-mirroring API; the
compute lives in ``libbcur_b200.so`` (sm_100a), reached through the C ABI in
``include/bcur_b200.h``.
"""

__all__ = ["bcur"]
