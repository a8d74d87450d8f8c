"""Oracle restatement of the reference ring arithmetic (ring.py) -- TEST ONLY.

Follows /root/reference/pkg/src/privtrain/ring.py:
  is_prime            ring.py:39-61   (deterministic Miller-Rabin)
  ntt_primes          ring.py:64-78   (descending p = 1 mod 2n below 2^bits)
  root_of_unity       ring.py:93-102  (smallest-witness primitive 2n-th root)
  NttPlan             ring.py:164-217 (CT forward natural->bit-reversed, GS inverse)
  sample_uniform      ring.py:292-302 (RingElem.random draw order)
  ring_mul_rns        ring.py:404-474 (per-prime NTT product; CRT is implicit in RNS)
  crt_combine         ring.py:477-491
  aux_primes / int_negacyclic_mul  ring.py:498-541
  ring_to_bytes / ring_from_bytes  ring.py:592-615
Polynomials are numpy arrays; NTTs are vectorised over leading batch axes.
"""
from __future__ import annotations

import struct

import numpy as np

_WITNESSES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    if n < 2:
        return False
    for w in _WITNESSES:
        if n % w == 0:
            return n == w
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for w in _WITNESSES:
        x = pow(w, d, n)
        if x == 1 or x == n - 1:
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def ntt_primes(n: int, bits: int, count: int, skip=()) -> list[int]:
    step = 2 * n
    cand = ((1 << bits) - 2) // step * step + 1
    out: list[int] = []
    skip = set(skip)
    while len(out) < count:
        if cand < step + 1:
            raise ValueError("prime supply exhausted")
        if cand not in skip and is_prime(cand):
            out.append(cand)
        cand -= step
    return out


def bitrev(x: int, bits: int) -> int:
    return int(format(x, f"0{bits}b")[::-1], 2) if bits else 0


def root_of_unity(order: int, p: int) -> int:
    cof = (p - 1) // order
    g = 2
    while g < p:
        psi = pow(g, cof, p)
        if pow(psi, order // 2, p) == p - 1:
            return psi
        g += 1
    raise ValueError(f"no order-{order} root mod {p}")


class NttPlan:
    """Per-(n, p) twiddles; same transform as ring._NttPlan (ring.py:164-217)."""

    _cache: dict = {}

    def __new__(cls, n: int, p: int):
        key = (n, p)
        if key not in cls._cache:
            obj = super().__new__(cls)
            obj._init(n, p)
            cls._cache[key] = obj
        return cls._cache[key]

    def _init(self, n: int, p: int):
        self.n, self.p = n, p
        self.logn = n.bit_length() - 1
        psi = root_of_unity(2 * n, p)
        self.small = p < (1 << 31)
        pw = [1] * n
        for i in range(1, n):
            pw[i] = pw[i - 1] * psi % p
        perm = [bitrev(i, self.logn) for i in range(n)]
        dt = np.uint64 if self.small else object
        self.w = np.array([pw[perm[i]] for i in range(n)], dtype=dt)
        self.n_inv = pow(n, -1, p)

    def _p(self):
        return np.uint64(self.p) if self.small else self.p

    def _cast(self, a):
        return np.asarray(a, dtype=np.uint64) if self.small else np.asarray(a, dtype=object)

    def forward(self, a: np.ndarray) -> np.ndarray:
        """Batched over leading axes; input canonical residues."""
        p = self._p()
        a = self._cast(a).copy()
        lead = a.shape[:-1]
        n = self.n
        half, m = n // 2, 1
        while half:
            v = a.reshape(*lead, m, 2 * half)
            z = self.w[m:2 * m].reshape(m, 1)
            x = v[..., :half].copy()
            y = v[..., half:] * z % p
            v[..., :half] = (x + y) % p
            v[..., half:] = (x + p - y) % p
            a = v.reshape(*lead, n)
            half //= 2
            m *= 2
        return a

    def inverse(self, a: np.ndarray) -> np.ndarray:
        p = self._p()
        a = self._cast(a).copy()
        lead = a.shape[:-1]
        n = self.n
        half, m = 1, n // 2
        while m:
            v = a.reshape(*lead, m, 2 * half)
            z = self.w[m:2 * m][::-1].reshape(m, 1)
            x = v[..., :half].copy()
            y = v[..., half:].copy()
            v[..., :half] = (x + y) % p
            v[..., half:] = (y + p - x) * z % p
            a = v.reshape(*lead, n)
            half *= 2
            m //= 2
        ninv = np.uint64(self.n_inv) if self.small else self.n_inv
        return a * ninv % p


def negacyclic_mul_mod(a: np.ndarray, b: np.ndarray, p: int) -> np.ndarray:
    """(a * b) mod (x^n + 1, p) for canonical residue arrays (batched)."""
    plan = NttPlan(a.shape[-1], p)
    fa = plan.forward(a)
    fb = plan.forward(b)
    pp = np.uint64(p) if plan.small else p
    return plan.inverse(fa * fb % pp)


def ring_mul_rns(a: np.ndarray, b: np.ndarray, primes) -> np.ndarray:
    """Residue-wise ring product, a/b shaped [..., L, N] (ring.py:462-474 per prime)."""
    out = np.empty(np.broadcast_shapes(a.shape, b.shape), dtype=np.uint64)
    for i, p in enumerate(primes):
        out[..., i, :] = np.asarray(negacyclic_mul_mod(a[..., i, :], b[..., i, :], p), dtype=np.uint64)
    return out


def to_rns(values, primes) -> np.ndarray:
    """Python ints (any sign) -> [L, N] residues."""
    vals = np.asarray(values, dtype=object)
    return np.stack([np.asarray(vals % p, dtype=np.uint64) for p in primes])


def crt_combine(residues: np.ndarray, primes) -> np.ndarray:
    """[L, ...] residues -> object ints in [0, prod) (ring.py:486-491)."""
    mod = 1
    for p in primes:
        mod *= p
    acc = np.zeros(residues.shape[1:], dtype=object)
    for r, p in zip(residues, primes):
        m = mod // p
        acc = acc + r.astype(object) * (m * pow(m, -1, p))
    return acc % mod


def centered(values, modulus: int) -> np.ndarray:
    v = np.asarray(values, dtype=object) % modulus
    return np.where(v > modulus // 2, v - modulus, v)


def sample_uniform(modulus: int, n: int, rng: np.random.Generator) -> np.ndarray:
    """RingElem.random (ring.py:292-302): uint64 draw when modulus < 2^63, else
    (bitlen+15)//8 little-endian random bytes per coefficient reduced mod q."""
    if modulus < (1 << 63):
        return rng.integers(0, modulus, size=n, dtype=np.uint64)
    nbytes = (modulus.bit_length() + 15) // 8
    return np.array([int.from_bytes(rng.bytes(nbytes), "little") % modulus for _ in range(n)], dtype=object)


_AUX: dict[int, list[int]] = {}


def aux_primes(n: int, need_bits: int) -> list[int]:
    """ring.py:502-513: 30-bit NTT primes until sum(bitlen-1) >= need_bits."""
    have = _AUX.setdefault(n, [])
    while sum(p.bit_length() - 1 for p in have) < need_bits:
        for p in ntt_primes(n, 30, len(have) + 1, skip=have):
            if p not in have:
                have.append(p)
    picked, tot = [], 0
    for p in have:
        picked.append(p)
        tot += p.bit_length() - 1
        if tot >= need_bits:
            break
    return picked


def int_negacyclic_mul(a, b, bound: int, n: int) -> np.ndarray:
    """Exact signed negacyclic product via aux-prime CRT (ring.py:516-541)."""
    primes = aux_primes(n, (2 * bound + 1).bit_length() + 1)
    ra = to_rns(a, primes)
    rb = to_rns(b, primes)
    res = np.stack([negacyclic_mul_mod(ra[i], rb[i], p) for i, p in enumerate(primes)])
    big = 1
    for p in primes:
        big *= p
    return centered(crt_combine(res, primes), big)


def limb_count(modulus: int) -> int:
    return max(1, (modulus.bit_length() + 63) // 64)


def ring_to_bytes(coeffs, n: int, modulus: int) -> bytes:
    """ring.py:592-599: <u32 n><u8 limbs> + per coefficient limbs x u64 LE positional."""
    limbs = limb_count(modulus)
    head = struct.pack("<IB", n, limbs)
    if limbs == 1:
        return head + np.asarray(coeffs, dtype=np.uint64).astype("<u8").tobytes()
    return head + b"".join(int(c).to_bytes(8 * limbs, "little") for c in coeffs)


def ring_from_bytes(data: bytes, n: int, modulus: int) -> np.ndarray:
    nn, limbs = struct.unpack_from("<IB", data, 0)
    assert nn == n and limbs == limb_count(modulus)
    if limbs == 1:
        return np.frombuffer(data, dtype="<u8", count=n, offset=5).astype(np.uint64) % np.uint64(modulus)
    w = 8 * limbs
    return np.array([int.from_bytes(data[5 + i * w: 5 + (i + 1) * w], "little") % modulus for i in range(n)],
                    dtype=object)
