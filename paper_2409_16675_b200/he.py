"""Device-resident mirror of privtrain.he (he.py): the BFV-style evaluator.

Same class and method names, argument meaning, noise algebra and errors as
the reference (he.py:34-531); ciphertexts stay in HBM as RNS residues
[parts, L, N] and every ring product runs in libctb200.so.  Client-side
randomness is drawn on the host with the reference's numpy calls in the
reference's order (keygen he.py:275-290, encrypt he.py:315-317), so the same
seeds give bit-identical keys and ciphertexts.

Extensions for the batched hot path (the reference loops one call at a time):
`CiphertextBatch`, `He.encrypt_many`, `He.decrypt_many`, `He.cp_mul_many`,
`He.cc_mul_many`; each ticks the meter once per logical operation, exactly as
the equivalent sequence of single calls would.

Only the "rlwe" backend exists here: the transparent "clear" backend is a
test stand-in of the reference, and the north star forbids multi-backend
dispatch on the device path.
"""
from __future__ import annotations

import dataclasses
import struct
import threading
import time
from typing import Sequence

import numpy as np
import torch

from . import _lib
from . import ring
from .device import BASE_Q, RnsContext, _ptr, _stream
from .params import (ACCUM_BUDGET, HeParams, default_cipher_params, default_he_params,  # noqa: F401
                     default_plain_params, p8192_he_params)
from .ring import RingElem, RingParams

__all__ = [
    "HeError", "PartCountError", "NoiseOverflowError", "BACKEND_CLEAR", "BACKEND_RLWE", "OPS", "ACCUM_BUDGET",
    "HeParams", "default_plain_params", "default_cipher_params", "default_he_params", "p8192_he_params",
    "OpMeter", "Ciphertext", "CiphertextBatch", "KeySet", "PublicKeys", "He",
]


class HeError(Exception):
    pass


class PartCountError(HeError):
    """A 3-part ciphertext reached an operation that needs 2 parts."""


class NoiseOverflowError(HeError):
    """The noise estimate exceeded the decryption budget."""


BACKEND_CLEAR = "clear"
BACKEND_RLWE = "rlwe"
OPS = ("CCMul", "CPMul", "CCAdd", "PPMul", "Relin", "Enc", "Dec")


# --------------------------------------------------------------------------- meters

class OpMeter:
    """Per-party, per-phase operation counters and cumulative wall time (he.py:173-208)."""

    def __init__(self):
        self._lock = threading.Lock()
        self.phase = "online"
        self.counts: dict[tuple[str, str], int] = {}
        self.seconds: dict[tuple[str, str], float] = {}

    def set_phase(self, phase: str):
        self.phase = phase

    def tick(self, op: str, secs: float = 0.0, count: int = 1):
        if count <= 0:
            return
        with self._lock:
            key = (self.phase, op)
            self.counts[key] = self.counts.get(key, 0) + count
            self.seconds[key] = self.seconds.get(key, 0.0) + secs

    def count(self, op: str, phase: str | None = None) -> int:
        with self._lock:
            if phase is None:
                return sum(v for (_, o), v in self.counts.items() if o == op)
            return self.counts.get((phase, op), 0)

    def time(self, op: str, phase: str | None = None) -> float:
        with self._lock:
            if phase is None:
                return sum(v for (_, o), v in self.seconds.items() if o == op)
            return self.seconds.get((phase, op), 0.0)

    def snapshot(self) -> dict:
        with self._lock:
            return {
                "counts": {f"{ph}:{op}": v for (ph, op), v in sorted(self.counts.items())},
                "seconds": {f"{ph}:{op}": v for (ph, op), v in sorted(self.seconds.items())},
            }


# --------------------------------------------------------------------------- ciphertexts and keys

class Ciphertext:
    """2 parts (fresh / after CPMul) or 3 parts (after raw CCMul); residues [parts, L, N] on device."""

    __slots__ = ("data", "noise_estimate", "backend_tag", "_cipher")

    def __init__(self, parts, noise_estimate: int, backend_tag: str, cipher: RingParams | None = None):
        if isinstance(parts, torch.Tensor):
            data = parts
            if cipher is None:
                raise HeError("a tensor-backed ciphertext needs its cipher ring")
        else:
            parts = tuple(parts)
            if len(parts) not in (2, 3):
                raise HeError(f"a ciphertext has 2 or 3 parts, not {len(parts)}")
            cipher = parts[0].params
            data = torch.stack([p.data for p in parts])
        if data.shape[0] not in (2, 3):
            raise HeError(f"a ciphertext has 2 or 3 parts, not {data.shape[0]}")
        self.data = data
        self.noise_estimate = int(noise_estimate)
        self.backend_tag = backend_tag
        self._cipher = cipher

    @property
    def nparts(self) -> int:
        return int(self.data.shape[0])

    @property
    def parts(self) -> tuple[RingElem, ...]:
        return tuple(RingElem(self._cipher, self.data[i]) for i in range(self.nparts))


class CiphertextBatch:
    """B ciphertexts with the same part count, residues [B, parts, L, N].

    Noise estimates are exact Python integers (he.py:103-132); a batch whose
    members share one estimate stores it once (`uniform_noise`)."""

    __slots__ = ("data", "_nu", "backend_tag", "_cipher", "eval_form")

    def __init__(self, data: torch.Tensor, noise, backend_tag: str, cipher: RingParams):
        self.data = data
        self.eval_form = None   # optional ctb_linear_addend form of `data` (server-side mask products)
        self._nu = int(noise) if isinstance(noise, int) else [int(v) for v in noise]
        self.backend_tag = backend_tag
        self._cipher = cipher

    @property
    def uniform_noise(self) -> int | None:
        return self._nu if isinstance(self._nu, int) else None

    @property
    def noise(self) -> list[int]:
        if isinstance(self._nu, int):
            return [self._nu] * int(self.data.shape[0])
        return self._nu

    def max_noise(self) -> int:
        return self._nu if isinstance(self._nu, int) else (max(self._nu) if self._nu else 0)

    @staticmethod
    def stack(cts: Sequence[Ciphertext]) -> "CiphertextBatch":
        if not cts:
            raise HeError("empty ciphertext batch")
        if len({c.nparts for c in cts}) != 1:
            raise PartCountError("ciphertexts in one batch must have the same part count")
        return CiphertextBatch(torch.stack([c.data for c in cts]), [c.noise_estimate for c in cts],
                               cts[0].backend_tag, cts[0]._cipher)

    def __len__(self):
        return int(self.data.shape[0])

    @property
    def nparts(self) -> int:
        return int(self.data.shape[1])

    def __getitem__(self, i) -> Ciphertext:
        nu = self._nu if isinstance(self._nu, int) else self._nu[i]
        return Ciphertext(self.data[i], nu, self.backend_tag, self._cipher)

    def unbind(self) -> list[Ciphertext]:
        return [self[i] for i in range(len(self))]


@dataclasses.dataclass(frozen=True)
class KeySet:
    """secret key stays client-side; public/relin keys go to the server (he.py:234-241)."""

    secret: RingElem | None
    public: tuple[RingElem, RingElem] | None
    relin: tuple[tuple[RingElem, RingElem], ...] | None
    backend_tag: str
    _prep: dict = dataclasses.field(default_factory=dict, compare=False, repr=False)


class PublicKeys:
    """The server-side subset of a KeySet."""

    def __init__(self, keys: KeySet):
        self.public = keys.public
        self.relin = keys.relin
        self.backend_tag = keys.backend_tag
        self._prep: dict = {}


def _prepared(keys, name: str, ctx: RnsContext, build) -> torch.Tensor:
    cache = keys._prep
    hit = cache.get(name)
    if hit is None:
        src = build()
        hit = torch.empty_like(src)
        npoly = src.numel() // (ctx.L * ctx.n)
        _lib.check(ctx._lib.ctb_prepare_operand(ctx._h, BASE_Q, _ptr(src), _ptr(hit), npoly, _stream()),
                   "ctb_prepare_operand")
        # built once and then read from any stream (concurrent jobs): complete it before publishing
        torch.cuda.current_stream().synchronize()
        cache[name] = hit
    return hit


# --------------------------------------------------------------------------- evaluator

class He:
    """One party's HE evaluator: parameters, backend, meter (he.py:258-518)."""

    def __init__(self, params: HeParams, backend: str = BACKEND_RLWE, meter: OpMeter | None = None,
                 sync_timing: bool = False):
        if backend not in (BACKEND_CLEAR, BACKEND_RLWE):
            raise ValueError(f"unknown backend {backend!r}")
        if backend == BACKEND_CLEAR:
            raise ValueError("the device path implements the 'rlwe' backend only (no multi-backend dispatch)")
        self.params = params
        self.backend = backend
        self.meter = meter or OpMeter()
        self.sync_timing = sync_timing
        cr, pr = params.cipher_ring, params.plain_ring
        self.ctx = RnsContext.get(params.n, cr.rns_primes, pr.rns_primes, params.relin_base_bits)
        self.L = self.ctx.L
        self._delta_res = [params.delta % p for p in self.ctx.q_primes]
        self._zero_plain = None
        self._draws: dict = {}

    # -- helpers --------------------------------------------------------------
    def _t0(self) -> float:
        if self.sync_timing:
            torch.cuda.synchronize()
        return time.perf_counter()

    def _elapsed(self, t0: float) -> float:
        if self.sync_timing:
            torch.cuda.synchronize()
        return time.perf_counter() - t0

    def _check_tag(self, ct):
        if ct.backend_tag != self.backend:
            raise HeError(f"ciphertext from backend {ct.backend_tag!r} fed to {self.backend!r}")

    def _small(self, vals: np.ndarray) -> torch.Tensor:
        """Small signed ints [k, N] -> residues [k, L, N]."""
        src = torch.from_numpy(np.ascontiguousarray(vals, dtype=np.int64)).cuda()
        k = src.shape[0]
        out = torch.empty((k, self.L, self.params.n), dtype=self.ctx.dtype(), device="cuda")
        _lib.check(self.ctx._lib.ctb_rns_from_small(self.ctx._h, BASE_Q, _ptr(src), _ptr(out), k, _stream()),
                   "ctb_rns_from_small")
        return out

    def _ternary(self, rng) -> np.ndarray:
        return rng.integers(-1, 2, size=self.params.n)

    def _error(self, rng) -> np.ndarray:
        bound = self.params.error_bound
        return np.clip(np.rint(rng.normal(0.0, self.params.noise_stddev, size=self.params.n)),
                       -bound, bound).astype(np.int64)

    def _rns(self, op: int, a: torch.Tensor, b: torch.Tensor | None, out: torch.Tensor | None = None):
        out = torch.empty_like(a) if out is None else out
        npoly = a.numel() // (self.L * self.params.n)
        _lib.check(self.ctx._lib.ctb_rns_elementwise(self.ctx._h, BASE_Q, op, _ptr(a), _ptr(b) if b is not None else None,
                                                     _ptr(out), npoly, _stream()), "ctb_rns_elementwise")
        return out

    def _plain_tensor(self, pts) -> torch.Tensor:
        if isinstance(pts, torch.Tensor):
            return pts.contiguous()
        for p in pts:
            if not p.params.compatible(self.params.plain_ring):
                raise HeError("plaintext must live in the plain ring")
        return torch.stack([p.data for p in pts]).contiguous()

    # -- keys -----------------------------------------------------------------
    def keygen(self, seed: int) -> KeySet:
        """he.py:272-290: draws s, a, e, then (a_i, e_i) per relinearisation digit."""
        rng = np.random.default_rng(seed)
        qr = self.params.cipher_ring
        s_vals = self._ternary(rng)
        a = RingElem.random(qr, rng)
        e_vals = self._error(rng)
        draws = []
        for _ in range(self.params.relin_digits):
            ai = RingElem.random(qr, rng)
            ei = self._error(rng)
            draws.append((ai, ei))
        small = self._small(np.stack([s_vals, e_vals] + [ei for _, ei in draws]))
        s, e = small[0], small[1]
        b = self._rns(2, self.ctx.ring_mul(a.data[None], s[None])[0], None)      # -(a s)
        b = self._rns(1, b, e)                                                    # -(a s) - e
        s2 = self.ctx.ring_mul(s[None], s[None])[0]
        D = self.params.relin_digits
        A = torch.stack([ai.data for ai, _ in draws])                             # [D, L, N]
        As = self.ctx.ring_mul(A, s[None])                                        # a_i s
        As = self._rns(0, As, small[2:2 + D])                                      # a_i s + e_i
        w = self.params.relin_base_bits
        shifts = torch.empty_like(A)
        for i in range(D):
            c = (1 << (w * i)) % self.params.q
            _lib.check(self.ctx._lib.ctb_rns_scalar_mul(self.ctx._h, BASE_Q, _ptr(s2),
                                                        _lib.u64_array([c % p for p in self.ctx.q_primes]),
                                                        _ptr(shifts[i]), 1, _stream()), "ctb_rns_scalar_mul")
        Bk = self._rns(1, shifts, As)                                             # s^2 2^(w i) - (a_i s + e_i)
        relin = tuple((RingElem(qr, Bk[i]), RingElem(qr, A[i])) for i in range(D))
        return KeySet(secret=RingElem(qr, s.clone()), public=(RingElem(qr, b), a), relin=relin,
                      backend_tag=self.backend)

    def _pk_prep(self, keys) -> torch.Tensor:
        return _prepared(keys, "pk", self.ctx, lambda: torch.stack([keys.public[0].data, keys.public[1].data]))

    # -- encrypt / decrypt ------------------------------------------------------
    def encrypt(self, m: RingElem, keys, rng: np.random.Generator) -> Ciphertext:
        """he.py:307-323: c0 = b u + e1 + Delta lift(m), c1 = a u + e2."""
        return self.encrypt_many([m], keys, rng)[0]

    def encrypt_many(self, ms, keys, rng) -> CiphertextBatch:
        """Encrypt plain polys (list of RingElem, an int64 tensor [B, N] of values in [0, t), or a
        packing.Gather descriptor: the packing fused into the encryption, ctb_encrypt_gather).

        With a numpy Generator the draws are the reference's, in the reference's
        order (identical to calling encrypt() B times).  With a torch.Generator
        on the device, u / e1 / e2 come from the same distributions (uniform
        ternary; rounded N(0, sigma^2) clipped to +-error_bound, he.py:292-303)
        drawn by the device Philox stream -- the production mode, which does not
        reproduce numpy's stream.
        """
        from . import packing
        t0 = self._t0()
        gather = ms if isinstance(ms, packing.Gather) else None
        if gather is not None:
            mt = None           # plaintexts read through the packing descriptor (ctb_encrypt_gather)
        elif isinstance(ms, torch.Tensor):
            mt = ms.contiguous()
        else:
            for m in ms:
                if not m.params.compatible(self.params.plain_ring):
                    raise HeError("payload must live in the plain ring")
            mt = self._plain_tensor(ms)
        B, n = (gather.n_polys if gather is not None else mt.shape[0]), self.params.n
        if self.params.error_bound > 127:
            raise HeError("the device encryptor takes int8 draws: error bound must be <= 127")
        if isinstance(rng, torch.Generator):
            draws = self._device_draws(B, rng)
        else:
            host = np.empty((B, 3, n), dtype=np.int8)
            for k in range(B):
                host[k, 0] = self._ternary(rng)
                host[k, 1] = self._error(rng)
                host[k, 2] = self._error(rng)
            nat = torch.from_numpy(host.reshape(B * 3, n)).cuda()
            draws = torch.empty_like(nat)
            _lib.check(self.ctx._lib.ctb_draws_from_natural(self.ctx._h, _ptr(nat), _ptr(draws), B, _stream()),
                       "ctb_draws_from_natural")
        pk = self._pk_prep(keys)
        out = torch.empty((B, 2, self.L, n), dtype=self.ctx.dtype(), device="cuda")
        if gather is not None:
            src = gather.src.contiguous()
            _lib.check(self.ctx._lib.ctb_encrypt_gather(
                self.ctx._h, _ptr(src) if src.numel() else None, src.numel(), _ptr(gather.maps), gather.maps.shape[0],
                _ptr(gather.kind), _ptr(gather.base), _ptr(draws.contiguous()), _ptr(pk), _ptr(out), B, _stream()),
                "ctb_encrypt_gather")
        else:
            _lib.check(self.ctx._lib.ctb_encrypt(self.ctx._h, _ptr(mt), _ptr(draws.contiguous()), _ptr(pk), _ptr(out),
                                                 B, _stream()), "ctb_encrypt")
        self.meter.tick("Enc", self._elapsed(t0), count=B)
        return CiphertextBatch(out, self.params.fresh_noise, self.backend, self.params.cipher_ring)

    def _device_draws(self, B: int, gen: torch.Generator) -> torch.Tensor:
        """int8 draws [B*3, N] from ctb_sample_draws, keyed by the generator's seed and
        Philox offset (advanced by B, so successive calls draw fresh values)."""
        out = self._draw_scratch(B * 3 * self.params.n).view(B * 3, self.params.n)
        seed = gen.initial_seed() & ((1 << 64) - 1)
        first = gen.get_offset()
        gen.set_offset(first + 4 * B)   # CUDA Philox offsets move in multiples of 4
        _lib.check(self.ctx._lib.ctb_sample_draws(self.ctx._h, seed, first, float(self.params.noise_stddev),
                                                  int(self.params.error_bound), _ptr(out), B, _stream()),
                   "ctb_sample_draws")
        return out

    def _draw_scratch(self, nbytes: int) -> torch.Tensor:
        """Per-evaluator int8 scratch for device draws, grown geometrically and reused (stream-ordered:
        every consumer of the draws is queued before the next encryption overwrites them).  A fresh
        sub-megabyte allocation per call occasionally cost tens of ms in the caching allocator's
        small-block pool (cudaMalloc of a new segment) inside cfg5's online phase."""
        key = torch.cuda.current_stream().cuda_stream   # one scratch per stream (concurrent jobs)
        buf = self._draws.get(key)
        if buf is None or buf.numel() < nbytes:
            size = 1 << max(20, (nbytes - 1).bit_length())
            buf = self._draws[key] = torch.empty(size, dtype=torch.int8, device="cuda")
        return buf[:nbytes]

    def _s_prep(self, keys, power: int) -> torch.Tensor:
        s = keys.secret.data
        if power == 1:
            return _prepared(keys, "s", self.ctx, lambda: s[None].contiguous())
        return _prepared(keys, f"s{power}", self.ctx,
                         lambda: self.ctx.ring_mul(s[None].contiguous(), s[None].contiguous()))

    def decrypt(self, ct: Ciphertext, keys: KeySet) -> RingElem:
        return self.decrypt_many([ct], keys)[0]

    def decrypt_many(self, cts, keys: KeySet) -> list[RingElem]:
        """he.py:329-351 over a batch: v = c0 + c1 s (+ c2 s^2); floor((v t + q//2)/q) mod t."""
        out = self.decrypt_values(cts, keys)
        return [RingElem(self.params.plain_ring, out[i]) for i in range(out.shape[0])]

    def _dec_acc(self, cts, keys: KeySet) -> tuple[CiphertextBatch, torch.Tensor]:
        """Noise gate (he.py:336-340) and v = c0 + c1 s (+ c2 s^2) residues [B, L, N]."""
        if isinstance(cts, CiphertextBatch):
            batch = cts
        else:
            for c in cts:
                self._check_tag(c)
            batch = CiphertextBatch.stack(list(cts))
        self._check_tag(batch)
        nu = batch.max_noise()
        if nu >= self.params.noise_budget:
            raise NoiseOverflowError(
                f"noise estimate 2^{nu.bit_length()} is at or above "
                f"the budget 2^{self.params.noise_budget.bit_length()}"
            )
        d = batch.data.contiguous()
        B, P = d.shape[0], d.shape[1]
        acc = torch.empty((B, self.L, self.params.n), dtype=d.dtype, device="cuda")
        # c0 + c1 s (+ c2 s^2) read in place from the [B][parts][L][N] batch (strided operands)
        _lib.check(self.ctx._lib.ctb_mul_prepared_strided(self.ctx._h, BASE_Q, _ptr(d[:, 1]), P,
                                                          _ptr(self._s_prep(keys, 1)), 0, _ptr(d[:, 0]), P,
                                                          _ptr(acc), B, _stream()), "ctb_mul_prepared_strided")
        if batch.nparts == 3:
            _lib.check(self.ctx._lib.ctb_mul_prepared_strided(self.ctx._h, BASE_Q, _ptr(d[:, 2]), P,
                                                              _ptr(self._s_prep(keys, 2)), 0, _ptr(acc), 1,
                                                              _ptr(acc), B, _stream()), "ctb_mul_prepared_strided")
        return batch, acc

    def decrypt_values(self, cts, keys: KeySet) -> torch.Tensor:
        """decrypt_many as one int64 tensor [B, N] of plain values (no per-poly objects)."""
        t0 = self._t0()
        batch, acc = self._dec_acc(cts, keys)
        out = torch.empty((len(batch), self.params.n), dtype=torch.int64, device="cuda")
        _lib.check(self.ctx._lib.ctb_decrypt_round(self.ctx._h, _ptr(acc), _ptr(out), len(batch), _stream()),
                   "ctb_decrypt_round")
        self.meter.tick("Dec", self._elapsed(t0), count=len(batch))
        return out

    def decrypt_extract(self, cts, keys: KeySet, out, sub: torch.Tensor | None = None,
                        centered: bool = True) -> torch.Tensor:
        """The client's tail of an online job in one epilogue: decrypt each slot, subtract the
        server's plain share p (linprot.py:444-450), extract the job's output tensor
        (packing.extract_output and friends) and centre it (to_signed_matrix) -- `out` is the job's
        packing.Scatter.  Only extracted coefficients are rounded (ctb_decrypt_round_extract)."""
        t0 = self._t0()
        batch, acc = self._dec_acc(cts, keys)
        if int(out.kind.shape[0]) != len(batch):
            raise HeError(f"extraction expects {int(out.kind.shape[0])} slots, got {len(batch)}")
        if sub is not None and tuple(sub.shape) != (len(batch), self.params.n):
            raise HeError("plain share shape does not match the slots")
        res = torch.empty(out.shape, dtype=torch.int64, device="cuda")   # the extraction covers every element
        _lib.check(self.ctx._lib.ctb_decrypt_round_extract(
            self.ctx._h, _ptr(acc), _ptr(sub.contiguous()) if sub is not None else None, _ptr(out.maps),
            out.maps.shape[0], _ptr(out.kind), _ptr(out.base), out.numel, int(centered), _ptr(res), len(batch),
            _stream()), "ctb_decrypt_round_extract")
        self.meter.tick("Dec", self._elapsed(t0), count=len(batch))
        return res

    # -- homomorphic ops --------------------------------------------------------
    def cc_add(self, a: Ciphertext, b: Ciphertext) -> Ciphertext:
        t0 = self._t0()
        self._check_tag(a)
        self._check_tag(b)
        if a.nparts != b.nparts:
            raise PartCountError(f"part counts differ: {a.nparts} vs {b.nparts}")
        ct = Ciphertext(self._rns(0, a.data, b.data), a.noise_estimate + b.noise_estimate, self.backend,
                        self.params.cipher_ring)
        self.meter.tick("CCAdd", self._elapsed(t0))
        return ct

    def cp_mul(self, ct: Ciphertext, pt: RingElem) -> Ciphertext:
        t0 = self._t0()
        self._check_tag(ct)
        if ct.nparts != 2:
            raise PartCountError("CPMul needs a 2-part ciphertext; relinearize first")
        if not pt.params.compatible(self.params.plain_ring):
            raise HeError("CPMul plaintext must live in the plain ring")
        out = self.ctx.cpmul(ct.data[None].contiguous(), pt.data[None].contiguous())[0]
        res = Ciphertext(out, self.params.cp_mul_noise(ct.noise_estimate), self.backend, self.params.cipher_ring)
        self.meter.tick("CPMul", self._elapsed(t0))
        return res

    def cp_mul_many(self, cts, pts) -> CiphertextBatch:
        """Batched CPMul: one fused kernel over all (ciphertext, plaintext) pairs."""
        t0 = self._t0()
        batch = cts if isinstance(cts, CiphertextBatch) else CiphertextBatch.stack(list(cts))
        self._check_tag(batch)
        if batch.nparts != 2:
            raise PartCountError("CPMul needs a 2-part ciphertext; relinearize first")
        out = self.ctx.cpmul(batch.data.contiguous(), self._plain_tensor(pts))
        u = batch.uniform_noise
        nu = self.params.cp_mul_noise(u) if u is not None else [self.params.cp_mul_noise(v) for v in batch.noise]
        res = CiphertextBatch(out, nu, self.backend, self.params.cipher_ring)
        self.meter.tick("CPMul", self._elapsed(t0), count=len(batch))
        return res

    def pp_mul(self, a: RingElem, b: RingElem) -> RingElem:
        t0 = self._t0()
        out = ring.ring_mul(a, b)
        self.meter.tick("PPMul", self._elapsed(t0))
        return out

    def cc_mul_raw(self, a: Ciphertext, b: Ciphertext) -> Ciphertext:
        """Tensor product only: 3 parts, not yet relinearised. Unmetered (he.py:384-407)."""
        return self.cc_mul_raw_many(CiphertextBatch.stack([a]), CiphertextBatch.stack([b]))[0]

    def cc_mul_raw_many(self, a: CiphertextBatch, b: CiphertextBatch) -> CiphertextBatch:
        from . import tensoring
        self._check_tag(a)
        self._check_tag(b)
        if a.nparts != 2 or b.nparts != 2:
            raise PartCountError("CCMul needs two 2-part ciphertexts")
        out = tensoring.tensor_round(self.ctx, a.data.contiguous(), b.data.contiguous())
        p = self.params
        if a.uniform_noise is not None and b.uniform_noise is not None:
            nu = 2 * p.n * p.t * (a.uniform_noise + b.uniform_noise) + 2 * p.n * p.n * p.t * p.t
        else:
            nu = [2 * p.n * p.t * (x + y) + 2 * p.n * p.n * p.t * p.t for x, y in zip(a.noise, b.noise)]
        return CiphertextBatch(out, nu, self.backend, p.cipher_ring)

    def _relin_prep(self, keys) -> torch.Tensor:
        def build():
            return torch.stack([torch.stack([bi.data, ai.data]) for bi, ai in keys.relin])  # [D, 2, L, N]
        return _prepared(keys, "relin", self.ctx, build)

    def relinearize(self, ct: Ciphertext, keys) -> Ciphertext:
        return self.relinearize_many(CiphertextBatch.stack([ct]), keys)[0]

    def relinearize_many(self, ct: CiphertextBatch, keys) -> CiphertextBatch:
        """he.py:409-432: (c0 + sum d_i b_i, c1 + sum d_i a_i), d_i the base-2^w digits of c2."""
        from . import tensoring
        t0 = self._t0()
        self._check_tag(ct)
        if ct.nparts != 3:
            raise PartCountError("relinearization expects a 3-part ciphertext")
        out = tensoring.relinearize(self.ctx, ct.data.contiguous(), self._relin_prep(keys))
        u = ct.uniform_noise
        nu = u + self.params.relin_noise if u is not None else [v + self.params.relin_noise for v in ct.noise]
        res = CiphertextBatch(out, nu, self.backend, self.params.cipher_ring)
        self.meter.tick("Relin", self._elapsed(t0), count=len(ct))
        return res

    def cc_mul(self, a: Ciphertext, b: Ciphertext, keys) -> Ciphertext:
        return self.cc_mul_many(CiphertextBatch.stack([a]), CiphertextBatch.stack([b]), keys)[0]

    def cc_mul_many(self, a: CiphertextBatch, b: CiphertextBatch, keys) -> CiphertextBatch:
        t0 = self._t0()
        out = self.relinearize_many(self.cc_mul_raw_many(a, b), keys)
        self.meter.tick("CCMul", self._elapsed(t0), count=len(a))
        return out

    # -- serialization ----------------------------------------------------------
    def ct_to_bytes(self, ct: Ciphertext) -> bytes:
        body = b"".join(ring.ring_to_bytes(p) for p in ct.parts)
        return struct.pack("<B", ct.nparts) + body

    def ct_from_bytes(self, data: bytes, noise: int | None = None) -> Ciphertext:
        (nparts,) = struct.unpack_from("<B", data, 0)
        rp = self.params.cipher_ring
        size = 5 + rp.n * 8 * rp.limb_count
        parts = []
        off = 1
        for _ in range(nparts):
            parts.append(ring.ring_from_bytes(data[off:off + size], rp))
            off += size
        nu = self._pessimistic_noise() if noise is None else noise
        return Ciphertext(parts, nu, self.backend)

    # -- batched wire format (one conversion kernel per batch) ------------------
    def batch_to_bytes(self, batch: CiphertextBatch) -> list[bytes]:
        """[ct_to_bytes(c) for c in batch], byte-identical, one rns->positional kernel."""
        B, k = len(batch), batch.nparts
        n = self.params.n
        limbs = self.params.cipher_ring.limb_count
        wc = self.ctx._lib.ctb_ctx_pos_words(self.ctx._h)
        words = torch.empty((B * k, n, wc), dtype=torch.int64, device="cuda")
        _lib.check(self.ctx._lib.ctb_rns_to_pos(self.ctx._h, _ptr(batch.data.contiguous()), _ptr(words), B * k,
                                                _stream()), "ctb_rns_to_pos")
        host = words.cpu().numpy().view("<u8")[:, :, :limbs]
        head = struct.pack("<IB", n, limbs)
        out = []
        for b in range(B):
            parts = [struct.pack("<B", k)]
            for j in range(k):
                parts.append(head)
                parts.append(np.ascontiguousarray(host[b * k + j]).tobytes())
            out.append(b"".join(parts))
        return out

    def batch_from_bytes(self, blobs: Sequence[bytes], noise: int | None = None) -> CiphertextBatch:
        """Inverse of batch_to_bytes / a list of ct_to_bytes blobs (ct_from_bytes, he.py:463-482)."""
        if not blobs:
            raise HeError("empty ciphertext batch")
        n = self.params.n
        limbs = self.params.cipher_ring.limb_count
        size = 5 + n * 8 * limbs
        k = blobs[0][0]
        body = np.empty((len(blobs) * k, n, limbs), dtype=np.uint64)
        for b, blob in enumerate(blobs):
            if blob[0] != k:
                raise PartCountError("ciphertexts in one batch must have the same part count")
            for j in range(k):
                off = 1 + j * size
                nn, lc = struct.unpack_from("<IB", blob, off)
                if nn != n or lc != limbs:
                    raise ring.RingError("serialized header does not match the ring parameters")
                body[b * k + j] = np.frombuffer(blob, dtype="<u8", count=n * limbs, offset=off + 5).reshape(n, limbs)
        wc = self.ctx._lib.ctb_ctx_pos_words(self.ctx._h)
        if wc != limbs:
            pad = np.zeros((body.shape[0], n, wc), dtype=np.uint64)
            pad[:, :, :min(wc, limbs)] = body[:, :, :min(wc, limbs)]
            body = pad
        words = torch.from_numpy(body.view(np.int64)).cuda()
        out = torch.empty((len(blobs), k, self.L, n), dtype=self.ctx.dtype(), device="cuda")
        _lib.check(self.ctx._lib.ctb_pos_to_rns(self.ctx._h, _ptr(words), _ptr(out), len(blobs) * k, _stream()),
                   "ctb_pos_to_rns")
        nu = self._pessimistic_noise() if noise is None else noise
        return CiphertextBatch(out, nu, self.backend, self.params.cipher_ring)

    def plain_to_bytes(self, polys: torch.Tensor) -> list[bytes]:
        """[ring_to_bytes(p) for p in polys] for plain-ring values [B, N] (one limb per coefficient)."""
        head = struct.pack("<IB", self.params.n, 1)
        host = polys.cpu().numpy().astype("<u8")
        return [head + host[i].tobytes() for i in range(host.shape[0])]

    def plain_from_bytes(self, blobs: Sequence[bytes]) -> torch.Tensor:
        n = self.params.n
        rows = []
        for blob in blobs:
            nn, lc = struct.unpack_from("<IB", blob, 0)
            if nn != n or lc != 1:
                raise ring.RingError("serialized header does not match the ring parameters")
            rows.append(np.frombuffer(blob, dtype="<u8", count=n, offset=5))
        host = (np.stack(rows) % np.uint64(self.params.t)).astype(np.int64)
        return torch.from_numpy(host).cuda()

    def _pessimistic_noise(self) -> int:
        p = self.params
        per_site = p.cc_mul_noise(p.fresh_noise, p.fresh_noise) + 2 * p.cp_mul_noise(p.fresh_noise)
        return per_site * ACCUM_BUDGET

    def public_keys_to_bytes(self, keys) -> bytes:
        blobs = [ring.ring_to_bytes(keys.public[0]), ring.ring_to_bytes(keys.public[1])]
        for b_i, a_i in keys.relin:
            blobs.append(ring.ring_to_bytes(b_i))
            blobs.append(ring.ring_to_bytes(a_i))
        return struct.pack("<H", len(blobs)) + b"".join(blobs)

    def public_keys_from_bytes(self, data: bytes) -> PublicKeys:
        (count,) = struct.unpack_from("<H", data, 0)
        rp = self.params.cipher_ring
        size = 5 + rp.n * 8 * rp.limb_count
        elems = []
        off = 2
        for _ in range(count):
            elems.append(ring.ring_from_bytes(data[off:off + size], rp))
            off += size
        public = (elems[0], elems[1])
        relin = tuple((elems[i], elems[i + 1]) for i in range(2, len(elems), 2))
        return PublicKeys(KeySet(None, public, relin, self.backend))

    def secret_key_to_bytes(self, keys: KeySet) -> bytes:
        if keys.secret is None:
            return b""
        return ring.ring_to_bytes(keys.secret)
