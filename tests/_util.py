import hashlib

import numpy as np


def digest(arr) -> str:
    """SHA-256 of a canonical little-endian uint64 array (matches make_golden.py)."""
    return hashlib.sha256(np.ascontiguousarray(np.asarray(arr, dtype=np.uint64), dtype="<u8").tobytes()).hexdigest()
