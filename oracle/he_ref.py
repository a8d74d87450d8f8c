"""Oracle restatement of the reference BFV-style scheme (he.py) -- TEST ONLY.

Cipher-ring polynomials are kept as RNS residues [parts, L, N] (uint64); the
reference keeps CRT-combined Python ints, which are congruent limb by limb,
so every residue here equals the reference's integer reduced mod q_i.

Follows /root/reference/pkg/src/privtrain/he.py:
  HeParamsRef + noise algebra    he.py:61-132
  default params                 he.py:135-165
  keygen / _ternary / _error     he.py:272-303
  encrypt / _lift                he.py:307-327
  decrypt                        he.py:329-351
  cp_mul                         he.py:366-382
  cc_mul_raw / _centered / _div_round   he.py:384-407, 521-531
  relinearize                    he.py:409-432
  pp_mul                         he.py:441-445 (ring.py:477-485 CRT)
"""
from __future__ import annotations

import dataclasses

import numpy as np

from . import ring_ref as R


@dataclasses.dataclass(frozen=True)
class HeParamsRef:
    n: int
    q_primes: tuple
    t_primes: tuple
    sigma: float = 3.2
    relin_base_bits: int = 16

    @property
    def q(self) -> int:
        out = 1
        for p in self.q_primes:
            out *= p
        return out

    @property
    def t(self) -> int:
        out = 1
        for p in self.t_primes:
            out *= p
        return out

    @property
    def L(self) -> int:
        return len(self.q_primes)

    @property
    def delta(self) -> int:
        return self.q // self.t

    @property
    def error_bound(self) -> int:
        return int(6 * self.sigma) + 1

    @property
    def relin_digits(self) -> int:
        w = self.relin_base_bits
        return (self.q.bit_length() + w - 1) // w

    # noise algebra, he.py:103-132
    @property
    def fresh_noise(self) -> int:
        return self.error_bound * (2 * self.n + 1)

    def cp_mul_noise(self, nu: int) -> int:
        return nu * self.n * (self.t // 2 + 1) + self.t * (self.n * self.t // 4 + 1)

    @property
    def relin_noise(self) -> int:
        return self.relin_digits * self.n * (1 << self.relin_base_bits) * self.error_bound

    def cc_mul_noise(self, a: int, b: int) -> int:
        n, t = self.n, self.t
        return 2 * n * t * (a + b) + 2 * n * n * t * t + self.relin_noise

    @property
    def noise_budget(self) -> int:
        return self.delta // 2

    def depth_ok(self, accum: int = 128) -> bool:
        worst = self.cc_mul_noise(self.fresh_noise, self.fresh_noise) + 2 * self.cp_mul_noise(self.fresh_noise)
        return worst * accum < self.noise_budget


def default_params(n: int = 4096, plain_bits: int = 25, plain_count: int = 2) -> HeParamsRef:
    """he.default_he_params (he.py:135-165): shortest 30-bit chain passing the budget."""
    tp = tuple(R.ntt_primes(n, plain_bits, plain_count))
    for count in range(3, 16):
        cand = HeParamsRef(n, tuple(R.ntt_primes(n, 30, count)), tp)
        if cand.depth_ok():
            return cand
    raise ValueError("no chain")


def p8192_params() -> HeParamsRef:
    """BASELINE P8192: q = 3 x 50-bit, t = 163841 * 147457."""
    return HeParamsRef(8192, tuple(R.ntt_primes(8192, 50, 3)), tuple(R.ntt_primes(8192, 18, 2)))


# ---------------------------------------------------------------- sampling

def ternary(p: HeParamsRef, rng) -> np.ndarray:
    return rng.integers(-1, 2, size=p.n)


def error(p: HeParamsRef, rng) -> np.ndarray:
    b = p.error_bound
    return np.clip(np.rint(rng.normal(0.0, p.sigma, size=p.n)), -b, b).astype(np.int64)


def small_to_rns(p: HeParamsRef, v) -> np.ndarray:
    v = np.asarray(v, dtype=np.int64)
    return np.stack([(v % np.int64(q)).astype(np.uint64) for q in p.q_primes])


def ints_to_rns(p: HeParamsRef, v) -> np.ndarray:
    return R.to_rns(v, p.q_primes)


def rns_to_ints(p: HeParamsRef, r: np.ndarray) -> np.ndarray:
    return R.crt_combine(np.asarray(r, dtype=np.uint64), p.q_primes)


def _add(p, a, b):
    qs = np.array(p.q_primes, dtype=np.uint64)[:, None]
    return (a + b) % qs


def _neg(p, a):
    qs = np.array(p.q_primes, dtype=np.uint64)[:, None]
    return (qs - a) % qs


def _mul(p, a, b):
    return R.ring_mul_rns(a, b, p.q_primes)


def keygen(p: HeParamsRef, seed: int) -> dict:
    """he.py:272-290 draw order: s, a, e, then (a_i, e_i) per digit."""
    rng = np.random.default_rng(seed)
    s = ternary(p, rng)
    a = ints_to_rns(p, R.sample_uniform(p.q, p.n, rng))
    e = error(p, rng)
    srns = small_to_rns(p, s)
    b = _neg(p, _add(p, _mul(p, a, srns), small_to_rns(p, e)))
    s2 = _mul(p, srns, srns)
    relin = []
    for i in range(p.relin_digits):
        ai = ints_to_rns(p, R.sample_uniform(p.q, p.n, rng))
        ei = error(p, rng)
        shift = (1 << (p.relin_base_bits * i))
        sh = np.stack([s2[j] * np.uint64(shift % q) % np.uint64(q) if q < (1 << 31)
                       else np.asarray(s2[j].astype(object) * (shift % q) % q, dtype=np.uint64)
                       for j, q in enumerate(p.q_primes)])
        qs = np.array(p.q_primes, dtype=np.uint64)[:, None]
        bi = (sh + qs - _add(p, _mul(p, ai, srns), small_to_rns(p, ei))) % qs
        relin.append((bi, ai))
    return {"s": s, "pk": (b, a), "relin": relin}


def lift(p: HeParamsRef, m) -> np.ndarray:
    """Centred lift of a plain payload into the cipher ring (he.py:325-327)."""
    m = np.asarray(m, dtype=np.uint64).astype(object)
    c = np.where(m > p.t // 2, m - p.t, m)
    return ints_to_rns(p, c)


def encrypt(p: HeParamsRef, m, pk, rng) -> np.ndarray:
    """he.py:307-323; draws u, e1, e2 in that order."""
    b, a = pk
    u = small_to_rns(p, ternary(p, rng))
    e1 = small_to_rns(p, error(p, rng))
    e2 = small_to_rns(p, error(p, rng))
    lm = lift(p, m)
    dm = np.stack([np.asarray(lm[j].astype(object) * (p.delta % q) % q, dtype=np.uint64)
                   for j, q in enumerate(p.q_primes)])
    c0 = _add(p, _add(p, _mul(p, b, u), e1), dm)
    c1 = _add(p, _mul(p, a, u), e2)
    return np.stack([c0, c1])


def decrypt(p: HeParamsRef, ct: np.ndarray, s) -> np.ndarray:
    """he.py:341-349: v = c0 + c1 s (+ c2 s^2), out = floor((v t + q//2) / q) mod t."""
    srns = small_to_rns(p, s)
    acc = ct[0]
    spow = srns
    for part in ct[1:]:
        acc = _add(p, acc, _mul(p, part, spow))
        spow = _mul(p, spow, srns)
    v = rns_to_ints(p, acc)
    q, t = p.q, p.t
    return np.array([(int(x) * t + q // 2) // q % t for x in v], dtype=np.uint64)


def cp_mul(p: HeParamsRef, ct: np.ndarray, pt) -> np.ndarray:
    """he.py:366-382: each part times the centred lift of pt."""
    lp = lift(p, pt)
    return np.stack([_mul(p, ct[0], lp), _mul(p, ct[1], lp)])


def div_round(a: int, b: int) -> int:
    """he.py:527-531: round(a/b), ties away from zero."""
    if a >= 0:
        return (a + b // 2) // b
    return -((-a + b // 2) // b)


def cc_mul_raw(p: HeParamsRef, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """he.py:384-407: exact tensor of centred lifts, then round(h t / q) mod q."""
    n, q, t = p.n, p.q, p.t
    bound = n * (q // 2 + 1) ** 2
    c0, c1 = (R.centered(rns_to_ints(p, part), q) for part in x)
    d0, d1 = (R.centered(rns_to_ints(p, part), q) for part in y)
    h0 = R.int_negacyclic_mul(c0, d0, bound, n)
    h1 = R.int_negacyclic_mul(c0, d1, bound, n) + R.int_negacyclic_mul(c1, d0, bound, n)
    h2 = R.int_negacyclic_mul(c1, d1, bound, n)
    parts = []
    for h in (h0, h1, h2):
        scaled = [div_round(int(v) * t, q) for v in h]
        parts.append(ints_to_rns(p, scaled))
    return np.stack(parts)


def relinearize(p: HeParamsRef, ct3: np.ndarray, relin) -> np.ndarray:
    """he.py:409-432: base-2^w digits of c2 (an integer in [0, q))."""
    w = p.relin_base_bits
    mask = (1 << w) - 1
    c2 = [int(v) for v in rns_to_ints(p, ct3[2])]
    acc0, acc1 = ct3[0], ct3[1]
    for i in range(p.relin_digits):
        d = small_to_rns(p, np.array([(v >> (w * i)) & mask for v in c2], dtype=np.int64))
        bi, ai = relin[i]
        acc0 = _add(p, acc0, _mul(p, d, bi))
        acc1 = _add(p, acc1, _mul(p, d, ai))
    return np.stack([acc0, acc1])


def cc_mul(p: HeParamsRef, x, y, relin) -> np.ndarray:
    return relinearize(p, cc_mul_raw(p, x, y), relin)


def pp_mul(p: HeParamsRef, a, b) -> np.ndarray:
    """Plain-ring product: per plain prime NTT product, then CRT (ring.py:477-491)."""
    a = np.asarray(a, dtype=np.uint64)
    b = np.asarray(b, dtype=np.uint64)
    res = np.stack([R.negacyclic_mul_mod(a % np.uint64(tp), b % np.uint64(tp), tp) for tp in p.t_primes])
    return np.asarray(R.crt_combine(res, p.t_primes), dtype=np.uint64)


def plain_add(p, a, b):
    return (np.asarray(a, dtype=np.uint64) + np.asarray(b, dtype=np.uint64)) % np.uint64(p.t)


def plain_sub(p, a, b):
    t = np.uint64(p.t)
    return (np.asarray(a, dtype=np.uint64) + (t - np.asarray(b, dtype=np.uint64))) % t
