"""Parameter objects and one-time host prime search for the device path.

Mirrors the reference's parameter layer so the same parameter sets come out:
  RingParams                ring.py:110-155 (degree, modulus, declared primes)
  is_prime / ntt_primes     ring.py:39-78   (deterministic Miller-Rabin, descending search)
  HeParams + noise algebra  he.py:61-132
  default_*_params          he.py:135-165
One deliberate extension: declared primes may be up to 50 bits (the reference
caps them below 2^31 for its numpy uint64 kernels, ring.py:134-135); the
device kernels carry 64-bit residues, which is what the N=8192 / 3 x 50-bit
configurations need.
"""
from __future__ import annotations

import dataclasses
from typing import Iterable

ACCUM_BUDGET = 128  # he.py:53

_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24 (covers every prime used here)."""
    if n < 2:
        return False
    for b in _MR_BASES:
        if n % b == 0:
            return n == b
    d, s = n - 1, 0
    while not d & 1:
        d >>= 1
        s += 1
    for b in _MR_BASES:
        x = pow(b, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def _is_pow2(n: int) -> bool:
    return n > 0 and n & (n - 1) == 0


def ntt_primes(n: int, bits: int, count: int, skip: Iterable[int] = ()) -> list[int]:
    """`count` distinct primes p = 1 (mod 2n) just below 2^bits, descending."""
    if not _is_pow2(n):
        raise ValueError("ring degree must be a power of two")
    step = 2 * n
    banned = set(skip)
    cand = ((1 << bits) - 2) // step * step + 1
    found: list[int] = []
    while len(found) < count:
        if cand <= step:
            raise ValueError(f"not enough {bits}-bit primes = 1 mod {step}")
        if cand not in banned and is_prime(cand):
            found.append(cand)
        cand -= step
    return found


@dataclasses.dataclass(frozen=True)
class RingParams:
    """Z_modulus[x]/(x^n + 1), optionally with a declared prime factorisation."""

    n: int
    modulus: int
    primes: tuple[int, ...] | None = None

    def __post_init__(self):
        if not _is_pow2(self.n):
            raise ValueError(f"ring degree {self.n} is not a power of two")
        if self.modulus <= 1:
            raise ValueError("modulus must exceed 1")
        if self.primes is not None:
            object.__setattr__(self, "primes", tuple(int(p) for p in self.primes))
            prod = 1
            for p in self.primes:
                if p % (2 * self.n) != 1:
                    raise ValueError(f"prime {p} is not 1 mod {2 * self.n}")
                if p >= 1 << 50:
                    raise ValueError(f"prime {p} too large for the device kernels (64-bit limbs: < 2^50)")
                prod *= p
            if prod != self.modulus:
                raise ValueError("declared primes do not multiply to the modulus")
            if len(set(self.primes)) != len(self.primes):
                raise ValueError("primes must be distinct")

    @property
    def ntt_enabled(self) -> bool:
        return self.modulus % (2 * self.n) == 1

    @property
    def limb_count(self) -> int:
        """64-bit words per coefficient on the wire (ring.py:147-148)."""
        return max(1, (self.modulus.bit_length() + 63) // 64)

    @property
    def uses_uint64(self) -> bool:
        return self.modulus < (1 << 63)

    @property
    def rns_primes(self) -> tuple[int, ...]:
        """Primes of the residue representation on device."""
        if self.primes is not None:
            return self.primes
        if is_prime(self.modulus) and self.ntt_enabled:
            return (self.modulus,)
        raise ValueError(f"modulus {self.modulus} has no NTT-friendly prime factorisation declared")

    def compatible(self, other: "RingParams") -> bool:
        return self.n == other.n and self.modulus == other.modulus


@dataclasses.dataclass(frozen=True)
class HeParams:
    """Cipher ring, plain ring, error width, relinearisation base (he.py:61-132)."""

    cipher_ring: RingParams
    plain_ring: RingParams
    noise_stddev: float = 3.2
    relin_base_bits: int = 16

    def __post_init__(self):
        if self.cipher_ring.n != self.plain_ring.n:
            raise ValueError("cipher and plain rings must share the degree")
        if self.cipher_ring.modulus <= self.plain_ring.modulus * 4:
            raise ValueError("ciphertext modulus must dominate the plain modulus")

    @property
    def n(self) -> int:
        return self.cipher_ring.n

    @property
    def q(self) -> int:
        return self.cipher_ring.modulus

    @property
    def t(self) -> int:
        return self.plain_ring.modulus

    @property
    def delta(self) -> int:
        return self.q // self.t

    @property
    def error_bound(self) -> int:
        return int(6 * self.noise_stddev) + 1

    @property
    def relin_digits(self) -> int:
        w = self.relin_base_bits
        return (self.q.bit_length() + w - 1) // w

    @property
    def fresh_noise(self) -> int:
        return self.error_bound * (2 * self.n + 1)

    def cp_mul_noise(self, nu: int) -> int:
        n, t = self.n, self.t
        return nu * n * (t // 2 + 1) + t * (n * t // 4 + 1)

    def cc_mul_noise(self, nu1: int, nu2: int) -> int:
        n, t = self.n, self.t
        return 2 * n * t * (nu1 + nu2) + 2 * n * n * t * t + self.relin_noise

    @property
    def relin_noise(self) -> int:
        return self.relin_digits * self.n * (1 << self.relin_base_bits) * self.error_bound

    @property
    def noise_budget(self) -> int:
        return self.delta // 2

    def check_depth_budget(self, accum: int = ACCUM_BUDGET):
        worst = self.cc_mul_noise(self.fresh_noise, self.fresh_noise) + 2 * self.cp_mul_noise(self.fresh_noise)
        if worst * accum >= self.noise_budget:
            raise ValueError(
                "parameters do not support one multiplication plus additions: "
                f"worst-case noise 2^{(worst * accum).bit_length()} vs budget "
                f"2^{self.noise_budget.bit_length()}"
            )


def _product(ps) -> int:
    out = 1
    for p in ps:
        out *= p
    return out


def default_plain_params(n: int = 4096, prime_bits: int = 25, primes: int = 2) -> RingParams:
    ps = ntt_primes(n, prime_bits, primes)
    return RingParams(n, _product(ps), primes=tuple(ps))


def default_cipher_params(n: int, plain_modulus: int, prime_bits: int = 30, accum: int = ACCUM_BUDGET) -> RingParams:
    """Shortest chain of `prime_bits` NTT primes that passes the depth budget."""
    for count in range(3, 16):
        ps = ntt_primes(n, prime_bits, count)
        cand = RingParams(n, _product(ps), primes=tuple(ps))
        try:
            HeParams(cand, RingParams(n, plain_modulus)).check_depth_budget(accum)
            return cand
        except ValueError:
            continue
    raise ValueError("no prime chain within 16 limbs satisfies the depth budget")


def default_he_params(n: int = 4096, plain: RingParams | None = None) -> HeParams:
    plain = plain or default_plain_params(n)
    params = HeParams(default_cipher_params(n, plain.modulus), plain)
    params.check_depth_budget()
    return params


def p8192_he_params() -> HeParams:
    """The BASELINE N=8192 set: q = 3 x 50-bit NTT primes, t = 163841 * 147457
    (SURVEY.md 8(d)); not expressible by the reference's he.He (ring.py:134)."""
    qs = ntt_primes(8192, 50, 3)
    ts = ntt_primes(8192, 18, 2)
    params = HeParams(RingParams(8192, _product(qs), tuple(qs)), RingParams(8192, _product(ts), tuple(ts)))
    params.check_depth_budget()
    return params
