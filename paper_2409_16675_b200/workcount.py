"""Algorithmic modular-multiplication counts of the hot-path steps (roofline accounting for bench.py).

Counted: the transform butterflies ((N/2) log2 N products per limb-transform) and the slotwise
products of the algorithm as this repository runs it.  Not counted: the exact
rounding / CRT / lift conversions and the additions, so achieved / peak is a LOWER bound on the
arithmetic utilisation.  Per-unit figures (N = 4096, L = 7 unless stated):

  CPMul (K2)                     L (5 NTT + 2 N)                         = 917,504   (N=8192, L=3: 847,872)
  encrypt one polynomial         L (3 NTT + 3 N)      NTT(u), b u, a u, 2 INTT, Delta m
  decrypt one slot               L (2 NTT + N)        c0 + c1 s (NTT(c1), product, INTT)
  online server (K3), per job    ciphertext parts 2 L (n_x + n_w) NTT, lifted masked plaintexts
                                 L (n_x + n_w)(NTT + N) and LT (n_x + n_w) NTT (plain side),
                                 per site 4 L N + LT N slotwise products, per slot (2 L + LT) INTT
  offline server (K4 + K5)       per distinct ciphertext 2 K NTT on the auxiliary base, per site
                                 4 K N products + 3 K INTT, per slot D L digit NTT + 2 D L N
                                 products + 2 L INTT
"""
from __future__ import annotations


def ntt(n: int) -> int:
    return (n // 2) * (n.bit_length() - 1)


def cpmul(n: int, L: int) -> int:
    return L * (5 * ntt(n) + 2 * n)


def encrypt(n: int, L: int, polys: int) -> int:
    return polys * L * (3 * ntt(n) + 3 * n)


def decrypt(n: int, L: int, slots: int) -> int:
    return slots * L * (2 * ntt(n) + n)


def online_server(n: int, L: int, LT: int, n_x: int, n_w: int, n_out: int, sites: int) -> int:
    polys = n_x + n_w
    return (2 * L * polys * ntt(n) + L * polys * (ntt(n) + n) + LT * polys * ntt(n)
            + sites * (4 * L * n + LT * n) + n_out * (2 * L + LT) * ntt(n))


def offline_server(n: int, L: int, K: int, D: int, n_x: int, n_w: int, n_out: int, sites: int) -> int:
    return (2 * K * (n_x + n_w) * ntt(n) + sites * (4 * K * n + 3 * K * ntt(n))
            + n_out * (D * L * ntt(n) + 2 * D * L * n + 2 * L * ntt(n)))


def online_job(n: int, L: int, LT: int, n_x: int, n_w: int, n_out: int, sites: int) -> int:
    """Client encrypt + server step + client decrypt of one (batched) online job."""
    return (encrypt(n, L, n_x + n_w) + online_server(n, L, LT, n_x, n_w, n_out, sites)
            + decrypt(n, L, n_out))


def offline_job(n: int, L: int, K: int, D: int, n_x: int, n_w: int, n_out: int, sites: int) -> int:
    """Client mask encryptions + the server's per-slot CCMul sums of one (batched) job."""
    return encrypt(n, L, n_x + n_w) + offline_server(n, L, K, D, n_x, n_w, n_out, sites)
