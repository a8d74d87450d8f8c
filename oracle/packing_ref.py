"""Oracle restatement of the reference's correlated packing (packing.py) -- TEST ONLY.

Follows /root/reference/pkg/src/privtrain/packing.py:
  window_feasible / tile_count / choose_tiles   packing.py:220-260
  _tile_positions / _axis_ownership            packing.py:272-307
  plan_correlated                              packing.py:310-337
  pack_input_correlated                        packing.py:407-426  (x[r0+i, c0+j] -> degree i*O + j)
  pack_kernel_correlated                       packing.py:429-445  (w[i, j] -> degree (h-1-i)*O + (h-1-j))
  extract_output (correlated)                  packing.py:476-509  (owned ranges, crop h-1-pad per side)
  FC packers                                   packing.py:541-605
and the job builders' site orders of linprot.py:108-257.  Plain numpy, values reduced mod t.
"""
from __future__ import annotations

import math

import numpy as np


def _product_degree(hw: int, ww: int, h: int) -> int:
    ow = max(ww, hw) + h - 1
    return (hw + h - 2) * ow + (ww + h - 2)


def window_feasible(H: int, W: int, h: int, hw: int, ww: int, n: int) -> bool:
    if not (h <= hw <= H and h <= ww <= W):
        return False
    ow = max(ww, hw) + h - 1
    return ww + hw * ow <= n and _product_degree(hw, ww, h) <= n - 1


def tile_count(H: int, W: int, h: int, hw: int, ww: int) -> int:
    rows = math.ceil((H - h + 1) / (hw - h + 1)) if hw > h - 1 else 0
    cols = math.ceil((W - h + 1) / (ww - h + 1)) if ww > h - 1 else 0
    return rows * cols


def choose_tiles(H: int, W: int, h: int, n: int) -> tuple[int, int]:
    best = None
    for hw in range(h, H + 1):
        for ww in range(h, W + 1):
            if not window_feasible(H, W, h, hw, ww, n):
                continue
            key = (tile_count(H, W, h, hw, ww), -(hw * ww), -hw)
            if best is None or key < best[0]:
                best = (key, (hw, ww))
    if best is None:
        raise ValueError("no feasible window")
    return best[1]


def _positions(extent: int, window: int, step: int) -> list[int]:
    if window >= extent:
        return [0]
    pos = list(range(0, extent - window, step)) + [extent - window]
    out = []
    for p in pos:
        if p not in out:
            out.append(p)
    return out


def _ownership(positions, window, kernel, full_extent):
    ranges, prev = [], 0
    for k, p0 in enumerate(positions):
        lo = 0 if k == 0 else max(p0 + kernel - 1, prev)
        hi = full_extent if k == len(positions) - 1 else p0 + window
        hi = max(hi, lo)
        ranges.append((lo, hi))
        prev = hi
    return ranges


def plan(H: int, W: int, h: int, pad: int, n: int) -> dict:
    """plan_correlated as a dict: tiles [(r0, c0)], owned [(u0, u1, v0, v1)], stride O, window."""
    hw, ww = choose_tiles(H, W, h, n)
    rows = _positions(H, hw, hw - h + 1)
    cols = _positions(W, ww, ww - h + 1)
    ro = _ownership(rows, hw, h, H + h - 1)
    co = _ownership(cols, ww, h, W + h - 1)
    tiles, owned = [], []
    for a, r0 in enumerate(rows):
        for b, c0 in enumerate(cols):
            tiles.append((r0, c0))
            owned.append(ro[a] + co[b])
    return {"H": H, "W": W, "h": h, "pad": pad, "n": n, "window": (hw, ww), "O": max(ww, hw) + h - 1,
            "tiles": tiles, "owned": owned}


def pack_input(x, pl: dict, t: int) -> np.ndarray:
    """x (H, W) -> [tiles, n] plain values in [0, t)."""
    x = np.asarray(x, dtype=np.int64)
    hw, ww = pl["window"]
    O, n = pl["O"], pl["n"]
    out = np.zeros((len(pl["tiles"]), n), dtype=np.int64)
    for k, (r0, c0) in enumerate(pl["tiles"]):
        sub = x[r0:r0 + hw, c0:c0 + ww]
        idx = (np.arange(sub.shape[0])[:, None] * O + np.arange(sub.shape[1])).ravel()
        out[k, idx] = sub.ravel()
    return (out % t).astype(np.uint64)


def pack_kernel(w, pl: dict, t: int) -> np.ndarray:
    w = np.asarray(w, dtype=np.int64)
    h, O, n = pl["h"], pl["O"], pl["n"]
    out = np.zeros(n, dtype=np.int64)
    r = h - 1 - np.arange(h)
    out[(r[:, None] * O + r).ravel()] = w.ravel()
    return (out % t).astype(np.uint64)


def extract(products: np.ndarray, pl: dict) -> np.ndarray:
    """[tiles, n] product coefficients (mod t) -> cropped [out_h, out_w] residues."""
    H, W, h, pad, O = pl["H"], pl["W"], pl["h"], pl["pad"], pl["O"]
    full = np.zeros((H + h - 1, W + h - 1), dtype=np.uint64)
    for (r0, c0), (u0, u1, v0, v1), poly in zip(pl["tiles"], pl["owned"], products):
        if u1 <= u0 or v1 <= v0:
            continue
        us = np.arange(u0, u1) - r0
        vs = np.arange(v0, v1) - c0
        full[u0:u1, v0:v1] = np.asarray(poly, dtype=np.uint64)[us[:, None] * O + vs]
    crop = h - 1 - pad
    if crop:
        full = full[crop:-crop, crop:-crop]
    return full


def centered(v, t: int) -> np.ndarray:
    v = np.asarray(v, dtype=np.int64) % np.int64(t)
    return np.where(v > t // 2, v - t, v)


# ---------------------------------------------------------------- job builders (linprot.py:108-257)

def conv_job(x, kernels, H, W, h, pad, n, t):
    """linprot.conv_job: x (cin, H, W), kernels (cout, cin, h, h); sites (c*T+t, co*cin+c, co*T+t)."""
    x = np.asarray(x, dtype=np.int64)
    kernels = np.asarray(kernels, dtype=np.int64)
    cout, cin = kernels.shape[:2]
    pl = plan(H, W, h, pad, n)
    T = len(pl["tiles"])
    xp = np.concatenate([pack_input(x[c], pl, t) for c in range(cin)])
    wp = np.stack([pack_kernel(kernels[co, c], pl, t) for co in range(cout) for c in range(cin)])
    sites = [(c * T + k, co * cin + c, co * T + k) for co in range(cout) for c in range(cin) for k in range(T)]

    def ext(out):
        return np.stack([extract(out[co * T:(co + 1) * T], pl) for co in range(cout)])

    return {"n_x": cin * T, "n_w": cout * cin, "n_out": cout * T, "sites": sites, "x": xp, "w": wp, "extract": ext}


def conv_grad_w_job(x, gy, H, W, h, pad, n, t):
    """linprot.conv_grad_w_job: out[co, ci] = conv(x[ci], gy[co]); sites (c*T+t, co, (co*cin+c)*T+t)."""
    x = np.asarray(x, dtype=np.int64)
    gy = np.asarray(gy, dtype=np.int64)
    cin, cout = x.shape[0], gy.shape[0]
    pl = plan(H, W, h, pad, n)
    T = len(pl["tiles"])
    xp = np.concatenate([pack_input(x[c], pl, t) for c in range(cin)])
    wp = np.stack([pack_kernel(gy[co], pl, t) for co in range(cout)])
    sites = [(c * T + k, co, (co * cin + c) * T + k) for co in range(cout) for c in range(cin) for k in range(T)]

    def ext(out):
        mats = [extract(out[s * T:(s + 1) * T], pl) for s in range(cout * cin)]
        side = mats[0].shape[-1]
        return np.stack(mats).reshape(cout, cin, side, side)

    return {"n_x": cin * T, "n_w": cout, "n_out": cout * cin * T, "sites": sites, "x": xp, "w": wp, "extract": ext}


def fc_job(x, w, n, t):
    """linprot.fc_job / packing.py:541-575: x at degree i; rows of W reversed at stride in_dim."""
    x = np.asarray(x, dtype=np.int64).ravel()
    w = np.asarray(w, dtype=np.int64)
    out_dim, in_dim = w.shape
    cap = max(1, n // in_dim)
    groups = math.ceil(out_dim / cap)
    xp = np.zeros((1, n), dtype=np.int64)
    xp[0, :in_dim] = x
    wp = np.zeros((groups, n), dtype=np.int64)
    for r in range(out_dim):
        g, k = divmod(r, cap)
        wp[g, k * in_dim:(k + 1) * in_dim] = w[r, ::-1]
    sites = [(0, j, j) for j in range(groups)]

    def ext(out):
        degs = np.arange(cap) * in_dim + in_dim - 1
        return np.concatenate([np.asarray(out[g], dtype=np.uint64)[degs] for g in range(groups)])[:out_dim]

    return {"n_x": 1, "n_w": groups, "n_out": groups, "sites": sites, "x": (xp % t).astype(np.uint64),
            "w": (wp % t).astype(np.uint64), "extract": ext}
