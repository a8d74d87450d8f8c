"""Device-resident mirror of privtrain.ring (ring.py) for the B200 hot path.

Same names, argument meaning and errors as the reference module
(ring.py:20-615); every arithmetic step runs in libctb200.so:

  * elements of rings with modulus < 2^63 (the plain ring t, single primes)
    hold an int64 CUDA tensor [N] of canonical values;
  * elements of larger rings (the cipher ring q = prod q_i) hold the RNS
    residues [L, N] (int32 words when every q_i < 2^30, else int64).

`RingElem.coeffs` materialises host values on demand (uint64 numpy array, or
an object array of Python ints for big moduli, exactly like the reference),
through the exact positional conversion kernel.

Deliberate differences: the degree must be >= 4 and <= 8192,
moduli must carry an NTT-friendly factorisation (the reference's schoolbook
fallback for non-NTT moduli, ring.py:427-439, has no device path and raises
NttUnavailableError), and declared primes may reach 50 bits.
"""
from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .device import BASE_Q, BASE_T, RnsContext, _ptr, _stream
from .params import RingParams, is_prime, ntt_primes  # noqa: F401  (re-exported like the reference)

__all__ = [
    "RingError", "ParamsMismatchError", "NttUnavailableError", "RingParams", "RingElem", "is_prime", "ntt_primes",
    "ring_add", "ring_sub", "ring_neg", "ring_scalar_mul", "ring_mul", "ntt_forward", "ntt_inverse",
    "pointwise_mul", "ring_to_bytes", "ring_from_bytes", "context_of",
]


class RingError(Exception):
    """Base error for ring arithmetic."""


class ParamsMismatchError(RingError):
    """Operands belong to different rings (or different domains)."""


class NttUnavailableError(RingError):
    """The modulus does not support a negacyclic NTT of this degree."""


# --------------------------------------------------------------------------- contexts

def context_of(params: RingParams) -> RnsContext:
    """Device context whose cipher base (and, for moduli < 2^63, plain base) is this ring."""
    try:
        primes = params.rns_primes
    except ValueError as exc:
        raise NttUnavailableError(str(exc)) from None
    small = params.uses_uint64 and len(primes) <= 2 and all(p < (1 << 30) for p in primes)
    return RnsContext.get(params.n, primes, primes if small else ())


def _is_small(params: RingParams) -> bool:
    return params.uses_uint64


def _check_pair(a: "RingElem", b: "RingElem", op: str):
    if not a.params.compatible(b.params):
        raise ParamsMismatchError(f"{op}: ring parameters differ")
    if a.domain != b.domain:
        raise ParamsMismatchError(f"{op}: domains differ ({a.domain} vs {b.domain})")


def _words_to_ints(words: np.ndarray) -> list[int]:
    """[N, W] little-endian uint64 words -> Python ints."""
    raw = np.ascontiguousarray(words, dtype="<u8").tobytes()
    w = words.shape[1] * 8
    return [int.from_bytes(raw[i * w:(i + 1) * w], "little") for i in range(words.shape[0])]


def _ints_to_words(values: Sequence[int], modulus: int, wcount: int) -> np.ndarray:
    w = wcount * 8
    raw = b"".join((int(v) % modulus).to_bytes(w, "little") for v in values)
    return np.frombuffer(raw, dtype="<u8").reshape(len(values), wcount).copy()


# --------------------------------------------------------------------------- elements

class RingElem:
    """Immutable element of Z_modulus[x]/(x^n + 1); coefficient of x^i at index i."""

    __slots__ = ("params", "domain", "data", "_host")

    def __init__(self, params: RingParams, data, domain: str = "coeff"):
        if isinstance(data, torch.Tensor):
            t = data
        else:  # host coefficient array: reduce like RingElem.from_ints
            t = RingElem.from_ints(params, data).data
        expect = (params.n,) if _is_small(params) else (len(params.rns_primes), params.n)
        if tuple(t.shape) != expect:
            raise RingError(f"expected {params.n} coefficients, got shape {tuple(t.shape)}")
        self.params = params
        self.domain = domain
        self.data = t
        self._host = None

    # construction ---------------------------------------------------------
    @staticmethod
    def zeros(params: RingParams) -> "RingElem":
        if _is_small(params):
            return RingElem(params, torch.zeros(params.n, dtype=torch.int64, device="cuda"))
        ctx = context_of(params)
        return RingElem(params, torch.zeros((ctx.L, params.n), dtype=ctx.dtype(), device="cuda"))

    @staticmethod
    def from_ints(params: RingParams, values) -> "RingElem":
        """Reduce arbitrary (possibly signed) integers into [0, modulus)."""
        arr = np.asarray(values)
        if arr.shape != (params.n,):
            raise RingError(f"expected {params.n} coefficients, got {arr.shape}")
        m = params.modulus
        small_ints = arr.dtype != object and arr.dtype.kind in "iu"
        if _is_small(params):
            if small_ints and arr.dtype != np.uint64:
                host = (arr.astype(np.int64) % np.int64(m)).astype(np.int64)
            elif small_ints:
                host = (arr % np.uint64(m)).astype(np.int64)
            else:
                host = np.array([int(v) % m for v in arr], dtype=np.int64)
            return RingElem(params, torch.from_numpy(host).cuda())
        ctx = context_of(params)
        out = torch.empty((ctx.L, params.n), dtype=ctx.dtype(), device="cuda")
        if small_ints and arr.dtype != np.uint64:
            src = torch.from_numpy(arr.astype(np.int64)).cuda()
            _lib.check(ctx._lib.ctb_rns_from_small(ctx._h, BASE_Q, _ptr(src), _ptr(out), 1, _stream()),
                       "ctb_rns_from_small")
            return RingElem(params, out)
        wc = ctx._lib.ctb_ctx_pos_words(ctx._h)
        words = torch.from_numpy(_ints_to_words(arr.tolist(), m, wc).view(np.int64)).cuda()
        _lib.check(ctx._lib.ctb_pos_to_rns(ctx._h, _ptr(words), _ptr(out), 1, _stream()), "ctb_pos_to_rns")
        return RingElem(params, out)

    @staticmethod
    def monomial(params: RingParams, coeff: int, degree: int) -> "RingElem":
        """coeff * x^degree with negacyclic degree reduction (x^n = -1)."""
        k, d = divmod(degree, params.n)
        if k % 2 == 1:
            coeff = -coeff
        vals = [0] * params.n
        vals[d] = coeff
        return RingElem.from_ints(params, np.array(vals, dtype=object))

    @staticmethod
    def random(params: RingParams, rng: np.random.Generator) -> "RingElem":
        """Same draws, same order as the reference (ring.py:292-302)."""
        if _is_small(params):
            arr = rng.integers(0, params.modulus, size=params.n, dtype=np.uint64)
            return RingElem(params, torch.from_numpy(arr.astype(np.int64)).cuda())
        nbytes = (params.modulus.bit_length() + 15) // 8
        ctx = context_of(params)
        wc = ctx._lib.ctb_ctx_pos_words(ctx._h)
        if nbytes % 4 == 0 and nbytes <= 8 * wc:
            # rng.bytes(k) n times == rng.bytes(k n) for k % 4 == 0; residues of the
            # unreduced integer equal those of its reduction mod q.
            raw = np.frombuffer(rng.bytes(nbytes * params.n), dtype=np.uint8).reshape(params.n, nbytes)
            buf = np.zeros((params.n, 8 * wc), dtype=np.uint8)
            buf[:, :nbytes] = raw
            words = torch.from_numpy(buf.view("<u8").view(np.int64).copy()).cuda()
            out = torch.empty((ctx.L, params.n), dtype=ctx.dtype(), device="cuda")
            _lib.check(ctx._lib.ctb_pos_to_rns(ctx._h, _ptr(words), _ptr(out), 1, _stream()), "ctb_pos_to_rns")
            return RingElem(params, out)
        vals = [int.from_bytes(rng.bytes(nbytes), "little") % params.modulus for _ in range(params.n)]
        return RingElem.from_ints(params, np.array(vals, dtype=object))

    # views ----------------------------------------------------------------
    @property
    def coeffs(self) -> np.ndarray:
        if self._host is None:
            if _is_small(self.params):
                host = self.data.cpu().numpy().astype(np.uint64)
            else:
                ctx = context_of(self.params)
                wc = ctx._lib.ctb_ctx_pos_words(ctx._h)
                words = torch.empty((self.params.n, wc), dtype=torch.int64, device="cuda")
                _lib.check(ctx._lib.ctb_rns_to_pos(ctx._h, _ptr(self.data), _ptr(words), 1, _stream()),
                           "ctb_rns_to_pos")
                host = np.array(_words_to_ints(words.cpu().numpy().view(np.uint64)), dtype=object)
            host.flags.writeable = False
            self._host = host
        return self._host

    def to_ints(self) -> list[int]:
        return [int(c) for c in self.coeffs]

    def to_signed(self) -> list[int]:
        m = self.params.modulus
        half = m // 2
        return [int(c) - m if int(c) > half else int(c) for c in self.coeffs]

    def is_zero(self) -> bool:
        return not bool(torch.any(self.data != 0))

    def __add__(self, other):
        return ring_add(self, other)

    def __sub__(self, other):
        return ring_sub(self, other)

    def __neg__(self):
        return ring_neg(self)

    def __mul__(self, other):
        if isinstance(other, RingElem):
            return ring_mul(self, other)
        return ring_scalar_mul(self, int(other))

    __rmul__ = __mul__

    def __eq__(self, other):
        return (isinstance(other, RingElem) and self.params.compatible(other.params)
                and self.domain == other.domain and bool(torch.equal(self.data, other.data)))

    def __hash__(self):
        return hash((self.params.n, self.params.modulus, self.domain, bytes(str(self.to_ints()), "ascii")))

    def __repr__(self):
        head = ", ".join(str(int(c)) for c in self.coeffs[:4])
        return f"RingElem(n={self.params.n}, mod={self.params.modulus}, [{head}, ...], {self.domain}, cuda)"


# --------------------------------------------------------------------------- arithmetic

def _values_to_rns(ctx: RnsContext, values: torch.Tensor) -> torch.Tensor:
    """[N] canonical values of a modulus < 2^63 -> [1, L, N] residues (exact positional conversion)."""
    wc = ctx._lib.ctb_ctx_pos_words(ctx._h)
    words = values.view(-1, 1)
    if wc != 1:
        words = torch.cat([words, torch.zeros((values.numel(), wc - 1), dtype=torch.int64, device=values.device)], 1)
    out = torch.empty((1, ctx.L, values.numel()), dtype=ctx.dtype(), device="cuda")
    _lib.check(ctx._lib.ctb_pos_to_rns(ctx._h, _ptr(words.contiguous()), _ptr(out), 1, _stream()), "ctb_pos_to_rns")
    return out


def _rns_to_values(ctx: RnsContext, res: torch.Tensor) -> torch.Tensor:
    wc = ctx._lib.ctb_ctx_pos_words(ctx._h)
    n = res.shape[-1]
    words = torch.empty((n, wc), dtype=torch.int64, device="cuda")
    _lib.check(ctx._lib.ctb_rns_to_pos(ctx._h, _ptr(res.contiguous()), _ptr(words), 1, _stream()), "ctb_rns_to_pos")
    return words[:, 0].contiguous()


def _as_residues(ctx: RnsContext, a: RingElem) -> torch.Tensor:
    """Value tensor of a ring with modulus < 2^63 viewed as [1, L, N] residues: a single prime
    (>= 2^30, so the context's words are 64-bit) is its own residue; several primes go through
    the exact positional conversion."""
    if ctx.L == 1:
        return a.data.view(1, 1, -1).to(ctx.dtype())
    return _values_to_rns(ctx, a.data)


def _from_residues(ctx: RnsContext, res: torch.Tensor) -> torch.Tensor:
    if ctx.L == 1:
        return res.reshape(-1).to(torch.int64)
    return _rns_to_values(ctx, res)


def _small_op(a: RingElem, b: RingElem | None, op: int, scalar: int = 0) -> RingElem:
    ctx = context_of(a.params)
    if ctx.t:  # plain-ring kernel (t = modulus)
        out = torch.empty_like(a.data)
        _lib.check(ctx._lib.ctb_plain_elementwise(ctx._h, op, _ptr(a.data), _ptr(b.data) if b is not None else None,
                                                  scalar, _ptr(out), 1, _stream()), "ctb_plain_elementwise")
        return RingElem(a.params, out, a.domain)
    # modulus < 2^63 whose factorisation is not a plain context (a prime >= 2^30, or 3+ primes):
    # run the RNS kernels on the residues and convert back
    x = _as_residues(ctx, a)
    out = torch.empty_like(x)
    if op == 3:
        _lib.check(ctx._lib.ctb_rns_scalar_mul(ctx._h, BASE_Q, _ptr(x), _lib.u64_array([scalar % p for p in ctx.q_primes]),
                                               _ptr(out), 1, _stream()), "ctb_rns_scalar_mul")
    else:
        y = _as_residues(ctx, b) if b is not None else None
        _lib.check(ctx._lib.ctb_rns_elementwise(ctx._h, BASE_Q, op, _ptr(x), _ptr(y) if y is not None else None,
                                                _ptr(out), 1, _stream()), "ctb_rns_elementwise")
    return RingElem(a.params, _from_residues(ctx, out), a.domain)


def _rns_op(a: RingElem, b: RingElem | None, op: int) -> RingElem:
    ctx = context_of(a.params)
    out = torch.empty_like(a.data)
    _lib.check(ctx._lib.ctb_rns_elementwise(ctx._h, BASE_Q, op, _ptr(a.data), _ptr(b.data) if b is not None else None,
                                            _ptr(out), 1, _stream()), "ctb_rns_elementwise")
    return RingElem(a.params, out, a.domain)


def ring_add(a: RingElem, b: RingElem) -> RingElem:
    """Coefficientwise (a + b) mod m (ring.py:363-370)."""
    _check_pair(a, b, "ring_add")
    return _small_op(a, b, 0) if _is_small(a.params) else _rns_op(a, b, 0)


def ring_sub(a: RingElem, b: RingElem) -> RingElem:
    _check_pair(a, b, "ring_sub")
    return _small_op(a, b, 1) if _is_small(a.params) else _rns_op(a, b, 1)


def ring_neg(a: RingElem) -> RingElem:
    return _small_op(a, None, 2) if _is_small(a.params) else _rns_op(a, None, 2)


def ring_scalar_mul(a: RingElem, c: int) -> RingElem:
    m = a.params.modulus
    c %= m
    if _is_small(a.params):
        return _small_op(a, None, 3, c)
    ctx = context_of(a.params)
    out = torch.empty_like(a.data)
    _lib.check(ctx._lib.ctb_rns_scalar_mul(ctx._h, BASE_Q, _ptr(a.data), _lib.u64_array([c % p for p in ctx.q_primes]),
                                           _ptr(out), 1, _stream()), "ctb_rns_scalar_mul")
    return RingElem(a.params, out, a.domain)


def ring_mul(a: RingElem, b: RingElem) -> RingElem:
    """Negacyclic product reduced mod (x^n + 1, modulus) (ring.py:404-427)."""
    _check_pair(a, b, "ring_mul")
    if a.domain == "eval":
        raise RingError("ring_mul expects coefficient-domain inputs; use pointwise_mul")
    ctx = context_of(a.params)
    if _is_small(a.params):
        if ctx.t:
            out = ctx.pp_mul(a.data.view(1, -1), b.data.view(1, -1)).view(-1)
            return RingElem(a.params, out)
        return RingElem(a.params, _from_residues(ctx, ctx.ring_mul(_as_residues(ctx, a), _as_residues(ctx, b))))
    out = ctx.ring_mul(a.data.unsqueeze(0), b.data.unsqueeze(0))
    return RingElem(a.params, out.squeeze(0))


def _single_prime(params: RingParams, what: str) -> RnsContext:
    if not params.ntt_enabled:
        raise NttUnavailableError(f"modulus {params.modulus} is not 1 mod {2 * params.n}")
    if not is_prime(params.modulus):
        raise NttUnavailableError(f"{what}: the evaluation domain is defined for a single NTT prime")
    return RnsContext.get(params.n, [params.modulus])


def ntt_forward(a: RingElem) -> RingElem:
    """Transform to the evaluation domain, bit-reversed order (ring.py:549-558)."""
    if a.domain != "coeff":
        raise RingError("ntt_forward expects a coefficient-domain element")
    ctx = _single_prime(a.params, "ntt_forward")
    x = a.data.view(1, 1, -1).to(ctx.dtype())
    return RingElem(a.params, ctx.ntt_forward(x).view(-1).to(torch.int64), domain="eval")


def ntt_inverse(a: RingElem) -> RingElem:
    if a.domain != "eval":
        raise RingError("ntt_inverse expects an evaluation-domain element")
    ctx = _single_prime(a.params, "ntt_inverse")
    x = a.data.view(1, 1, -1).to(ctx.dtype())
    return RingElem(a.params, ctx.ntt_inverse(x).view(-1).to(torch.int64), domain="coeff")


def pointwise_mul(a: RingElem, b: RingElem) -> RingElem:
    """Slotwise product of two evaluation-domain elements (ring.py:572-584)."""
    _check_pair(a, b, "pointwise_mul")
    if a.domain != "eval":
        raise RingError("pointwise_mul expects evaluation-domain elements")
    ctx = _single_prime(a.params, "pointwise_mul")
    x = a.data.view(1, 1, -1).to(ctx.dtype())
    y = b.data.view(1, 1, -1).to(ctx.dtype())
    return RingElem(a.params, ctx.pointwise_mul(x, y).view(-1).to(torch.int64), domain="eval")


# --------------------------------------------------------------------------- serialization
# n (u32 LE) | limb count (u8) | coefficient-major LE u64 limbs  (ring.py:588-615)

def ring_to_bytes(a: RingElem) -> bytes:
    import struct
    params = a.params
    limbs = params.limb_count
    head = struct.pack("<IB", params.n, limbs)
    if limbs == 1:
        return head + a.data.cpu().numpy().astype("<u8").tobytes()
    ctx = context_of(params)
    wc = ctx._lib.ctb_ctx_pos_words(ctx._h)
    words = torch.empty((params.n, wc), dtype=torch.int64, device="cuda")
    _lib.check(ctx._lib.ctb_rns_to_pos(ctx._h, _ptr(a.data), _ptr(words), 1, _stream()), "ctb_rns_to_pos")
    host = words.cpu().numpy().view("<u8")
    if wc != limbs:
        host = host[:, :limbs]
    return head + np.ascontiguousarray(host).tobytes()


def ring_from_bytes(data: bytes, params: RingParams) -> RingElem:
    import struct
    n, limbs = struct.unpack_from("<IB", data, 0)
    if n != params.n or limbs != params.limb_count:
        raise RingError("serialized header does not match the ring parameters")
    if limbs == 1:
        arr = np.frombuffer(data, dtype="<u8", count=n, offset=5).astype(np.uint64)
        return RingElem.from_ints(params, arr)
    ctx = context_of(params)
    wc = ctx._lib.ctb_ctx_pos_words(ctx._h)
    body = np.frombuffer(data, dtype="<u8", count=n * limbs, offset=5).reshape(n, limbs)
    if wc != limbs:
        pad = np.zeros((n, wc), dtype=np.uint64)
        pad[:, :min(wc, limbs)] = body[:, :min(wc, limbs)]
        body = pad
    words = torch.from_numpy(np.array(body, dtype=np.uint64).view(np.int64)).cuda()
    out = torch.empty((ctx.L, params.n), dtype=ctx.dtype(), device="cuda")
    _lib.check(ctx._lib.ctb_pos_to_rns(ctx._h, _ptr(words), _ptr(out), 1, _stream()), "ctb_pos_to_rns")
    return RingElem(params, out)


def ring_mul_schoolbook(a: RingElem, b: RingElem) -> RingElem:
    """The reference keeps an O(n^2) oracle (ring.py:430-439); on this path the
    independent oracle lives in oracle/ (test infrastructure), so this raises."""
    raise NttUnavailableError("schoolbook multiplication is not part of the device path (see oracle/)")
