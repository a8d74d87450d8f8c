"""Independent plaintext convolution oracle -- TEST ONLY.

Restates the reference's tests/oracles.py:14-35 (direct sliding-window
cross-correlation with zero padding, exact in int64), extended to channels.
"""
import numpy as np


def conv2d(x, w, pad: int) -> np.ndarray:
    x = np.asarray(x, dtype=np.int64)
    w = np.asarray(w, dtype=np.int64)
    h = w.shape[0]
    xp = np.pad(x, pad)
    win = np.lib.stride_tricks.sliding_window_view(xp, (h, h))
    return np.einsum("uvab,ab->uv", win, w)


def conv2d_multi(x, w, pad: int) -> np.ndarray:
    """x (cin, H, W), w (cout, cin, h, h) -> (cout, H', W')."""
    x = np.asarray(x, dtype=np.int64)
    w = np.asarray(w, dtype=np.int64)
    return np.stack([sum(conv2d(x[c], w[o, c], pad) for c in range(x.shape[0])) for o in range(w.shape[0])])
