"""Device-resident RNS contexts: the Python face of the C ABI.

PyTorch supplies device memory and the current CUDA stream (plumbing only);
every arithmetic step runs in libctb200.so.  Residue tensors are
[poly][limb][N] with dtype int32 for bases whose primes are < 2^30 (the words
are the unsigned residues, all < 2^30) and int64 otherwise; plain-ring
polynomials are int64 [poly][N] with values in [0, t).
"""
from __future__ import annotations

import ctypes
import threading

import torch

from . import _lib
from ._lib import BASE_B, BASE_Q, BASE_T, check

__all__ = ["RnsContext", "BASE_Q", "BASE_T", "BASE_B"]


def _stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


class RnsContext:
    """Tables for one (N, q primes, t primes) parameter set; read-only, thread-safe."""

    _cache: dict = {}
    _cache_lock = threading.Lock()

    @classmethod
    def get(cls, n: int, q_primes, t_primes=(), relin_base_bits: int = 16, device=None) -> "RnsContext":
        dev = torch.cuda.current_device() if device is None else torch.device(device).index
        key = (n, tuple(int(p) for p in q_primes), tuple(int(p) for p in t_primes), relin_base_bits, dev)
        with cls._cache_lock:
            ctx = cls._cache.get(key)
            if ctx is None:
                ctx = cls(n, key[1], key[2], relin_base_bits)
                cls._cache[key] = ctx
        return ctx

    def __init__(self, n: int, q_primes, t_primes=(), relin_base_bits: int = 16):
        if not torch.cuda.is_available():
            raise _lib.CtbError(_lib.CTB_ERR_CUDA, "RnsContext", "no CUDA device visible (no CPU fallback exists)")
        self._lib = _lib.load()
        self.n = int(n)
        self.q_primes = tuple(int(p) for p in q_primes)
        self.t_primes = tuple(int(p) for p in t_primes)
        self.device = torch.device("cuda", torch.cuda.current_device())
        h = ctypes.c_void_p()
        q = _lib.u64_array(self.q_primes)
        t = _lib.u64_array(self.t_primes)
        check(self._lib.ctb_ctx_create(ctypes.byref(h), self.n, q, len(self.q_primes), t, len(self.t_primes),
                                       relin_base_bits), "ctb_ctx_create")
        self._h = h
        self.t = 0
        if self.t_primes:
            self.t = 1
            for p in self.t_primes:
                self.t *= p

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.ctb_ctx_destroy(h)
            except Exception:
                pass

    # -- introspection ------------------------------------------------------
    def word_bytes(self, base: int = BASE_Q) -> int:
        return self._lib.ctb_ctx_word_bytes(self._h, base)

    def base_size(self, base: int = BASE_Q) -> int:
        return self._lib.ctb_ctx_base_size(self._h, base)

    def dtype(self, base: int = BASE_Q) -> torch.dtype:
        return torch.int32 if self.word_bytes(base) == 4 else torch.int64

    @property
    def L(self) -> int:
        return len(self.q_primes)

    # -- checks ---------------------------------------------------------------
    def _check_res(self, x: torch.Tensor, base: int, name: str) -> int:
        if not (x.is_cuda and x.is_contiguous()):
            raise ValueError(f"{name}: expected a contiguous CUDA tensor")
        if x.dtype != self.dtype(base):
            raise ValueError(f"{name}: expected dtype {self.dtype(base)}, got {x.dtype}")
        L = self.base_size(base)
        if x.dim() < 2 or x.shape[-1] != self.n or x.shape[-2] != L:
            raise ValueError(f"{name}: expected [..., {L}, {self.n}], got {tuple(x.shape)}")
        return x.numel() // (L * self.n)

    def _check_plain(self, x: torch.Tensor, name: str) -> int:
        if not (x.is_cuda and x.is_contiguous()) or x.dtype != torch.int64 or x.shape[-1] != self.n:
            raise ValueError(f"{name}: expected a contiguous CUDA int64 tensor [..., {self.n}]")
        return x.numel() // self.n

    # -- kernels ----------------------------------------------------------------
    def ntt_forward(self, x: torch.Tensor, base: int = BASE_Q, out: torch.Tensor | None = None) -> torch.Tensor:
        npoly = self._check_res(x, base, "ntt_forward")
        out = torch.empty_like(x) if out is None else out
        check(self._lib.ctb_ntt_forward(self._h, base, _ptr(x), _ptr(out), npoly, _stream()), "ctb_ntt_forward")
        return out

    def ntt_inverse(self, x: torch.Tensor, base: int = BASE_Q, out: torch.Tensor | None = None) -> torch.Tensor:
        npoly = self._check_res(x, base, "ntt_inverse")
        out = torch.empty_like(x) if out is None else out
        check(self._lib.ctb_ntt_inverse(self._h, base, _ptr(x), _ptr(out), npoly, _stream()), "ctb_ntt_inverse")
        return out

    def pointwise_mul(self, a: torch.Tensor, b: torch.Tensor, base: int = BASE_Q) -> torch.Tensor:
        npoly = self._check_res(a, base, "pointwise_mul")
        if b.shape != a.shape:
            raise ValueError("pointwise_mul: shape mismatch")
        self._check_res(b, base, "pointwise_mul")
        out = torch.empty_like(a)
        check(self._lib.ctb_pointwise_mul(self._h, base, _ptr(a), _ptr(b), _ptr(out), npoly, _stream()),
              "ctb_pointwise_mul")
        return out

    def ring_mul(self, a: torch.Tensor, b: torch.Tensor, base: int = BASE_Q) -> torch.Tensor:
        """Negacyclic products a[i] * b[i]; a leading dim of 1 broadcasts."""
        na = self._check_res(a, base, "ring_mul")
        nb = self._check_res(b, base, "ring_mul")
        n = max(na, nb)
        if na not in (1, n) or nb not in (1, n):
            raise ValueError("ring_mul: batch sizes do not broadcast")
        shape = a.shape if na == n else b.shape
        out = torch.empty(shape, dtype=a.dtype, device=a.device)
        check(self._lib.ctb_ring_mul(self._h, base, _ptr(a), 0 if na == 1 else 1, _ptr(b), 0 if nb == 1 else 1,
                                     _ptr(out), n, _stream()), "ctb_ring_mul")
        return out

    def cpmul(self, ct: torch.Tensor, pt: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """ct [B, 2, L, N] x pt [B, N] (int64 in [0, t)) -> [B, 2, L, N]."""
        if ct.dim() != 4 or ct.shape[1] != 2:
            raise ValueError("cpmul: ciphertexts must be [B, 2, L, N]")
        self._check_res(ct, BASE_Q, "cpmul")
        nb = self._check_plain(pt, "cpmul")
        if nb != ct.shape[0]:
            raise ValueError("cpmul: one plaintext per ciphertext")
        out = torch.empty_like(ct) if out is None else out
        check(self._lib.ctb_cpmul(self._h, _ptr(ct), _ptr(pt), _ptr(out), ct.shape[0], _stream()), "ctb_cpmul")
        return out

    def cpmul_host(self, ct_h: torch.Tensor, pt_h: torch.Tensor, out_h: torch.Tensor, chunks: int = 16,
                   slots: int = 3) -> None:
        """CPMul of host-resident (pinned) batches: chunked H2D / k_cpmul / D2H on three
        streams so both copy directions overlap each other and the kernel.  Returns
        after enqueueing; the caller synchronises (or records an event on the
        current stream, which is made to wait for the last D2H)."""
        B = ct_h.shape[0]
        if B == 0:
            return
        step = -(-B // max(1, chunks))
        cur = torch.cuda.current_stream()
        # streams and staging buffers are per calling thread (contexts are shared by the two
        # party threads of an in-process session, RnsContext.get)
        tl = self.__dict__.setdefault("_pipe_tls", threading.local())
        if not hasattr(tl, "streams"):
            tl.streams = [torch.cuda.Stream() for _ in range(3)]
            tl.key = None
        s_in, s_comp, s_out = tl.streams
        shape_ct = (step,) + tuple(ct_h.shape[1:])
        key = (shape_ct, ct_h.dtype, pt_h.shape[1:], slots)
        if tl.key != key:
            tl.buf = [(torch.empty(shape_ct, dtype=ct_h.dtype, device="cuda"),
                       torch.empty((step,) + tuple(pt_h.shape[1:]), dtype=pt_h.dtype, device="cuda"),
                       torch.empty(shape_ct, dtype=ct_h.dtype, device="cuda")) for _ in range(slots)]
            tl.key = key
        ev_in = [torch.cuda.Event() for _ in range(slots)]
        ev_comp = [torch.cuda.Event() for _ in range(slots)]
        ev_out = [None] * slots
        start = torch.cuda.Event()
        start.record(cur)
        for s in (s_in, s_comp, s_out):
            s.wait_event(start)
        for i, lo in enumerate(range(0, B, step)):
            hi = min(B, lo + step)
            n = hi - lo
            k = i % slots
            ct_d, pt_d, out_d = tl.buf[k]
            if ev_out[k] is not None:
                s_in.wait_event(ev_out[k])
            with torch.cuda.stream(s_in):
                ct_d[:n].copy_(ct_h[lo:hi], non_blocking=True)
                pt_d[:n].copy_(pt_h[lo:hi], non_blocking=True)
            ev_in[k].record(s_in)
            s_comp.wait_event(ev_in[k])
            with torch.cuda.stream(s_comp):
                self.cpmul(ct_d[:n], pt_d[:n], out=out_d[:n])
            ev_comp[k].record(s_comp)
            s_out.wait_event(ev_comp[k])
            with torch.cuda.stream(s_out):
                out_h[lo:hi].copy_(out_d[:n], non_blocking=True)
            ev_out[k] = torch.cuda.Event()
            ev_out[k].record(s_out)
        cur.wait_stream(s_out)

    # -- dense bit-packed transfer format (ctb_bits_pack / ctb_bits_unpack) -------------------
    @property
    def q_bits(self) -> int:
        """Bits per cipher residue in the packed format (30 for the default 30-bit chain)."""
        return max(int(p).bit_length() for p in self.q_primes)

    @property
    def t_bits(self) -> int:
        return int(self.t).bit_length()

    def pack_bits(self, x: torch.Tensor, bits: int, out: torch.Tensor | None = None) -> torch.Tensor:
        """Values of x (uint32-width int32 or int64 words, each < 2^bits) -> packed int32 words."""
        word = x.element_size()
        words = int(self._lib.ctb_bits_words(bits, x.numel()))
        out = torch.empty(words, dtype=torch.int32, device="cuda") if out is None else out
        check(self._lib.ctb_bits_pack(self._h, word, _ptr(x.contiguous()), bits, _ptr(out), x.numel(), _stream()),
              "ctb_bits_pack")
        return out

    def unpack_bits(self, packed: torch.Tensor, bits: int, shape, dtype, out: torch.Tensor | None = None) -> torch.Tensor:
        count = 1
        for d in shape:
            count *= int(d)
        out = torch.empty(tuple(shape), dtype=dtype, device="cuda") if out is None else out
        check(self._lib.ctb_bits_unpack(self._h, out.element_size(), _ptr(packed), bits, _ptr(out), count, _stream()),
              "ctb_bits_unpack")
        return out

    def cpmul_host_packed(self, ctp_h: torch.Tensor, ptp_h: torch.Tensor, outp_h: torch.Tensor, batch: int,
                          chunks: int = 16, slots: int = 3) -> None:
        """cpmul_host over the dense packed transfer format: ctp_h holds the batch's residues as
        q_bits-bit values ([batch][2][L][N] order, pack_bits), ptp_h the plaintexts as t_bits-bit
        values, outp_h receives the products packed like ctp_h (all pinned int32 word tensors).
        Per chunk: H2D of the packed words, unpack + k_cpmul + pack on the device, D2H -- 30-bit
        residues cross PCIe at 3.75 B and 50-bit plaintexts at 6.25 B instead of 4 B / 8 B."""
        if batch == 0:
            return
        L, n = self.L, self.n
        qb, tb = self.q_bits, self.t_bits
        per_ct = 2 * L * n * qb // 32        # words per ciphertext (whole words: n * bits % 32 == 0)
        per_pt = n * tb // 32
        if (2 * L * n * qb) % 32 or (n * tb) % 32:
            raise ValueError("cpmul_host_packed: ring degree too small for word-aligned items")
        step = -(-batch // max(1, chunks))
        cur = torch.cuda.current_stream()
        tl = self.__dict__.setdefault("_pipe_tls_packed", threading.local())
        if not hasattr(tl, "streams"):
            tl.streams = [torch.cuda.Stream() for _ in range(3)]
            tl.key = None
        s_in, s_comp, s_out = tl.streams
        key = (step, slots)
        if tl.key != key:
            dt = self.dtype()
            tl.buf = [(torch.empty(step * per_ct, dtype=torch.int32, device="cuda"),
                       torch.empty(step * per_pt, dtype=torch.int32, device="cuda"),
                       torch.empty((step, 2, L, n), dtype=dt, device="cuda"),
                       torch.empty((step, n), dtype=torch.int64, device="cuda"),
                       torch.empty((step, 2, L, n), dtype=dt, device="cuda"),
                       torch.empty(step * per_ct, dtype=torch.int32, device="cuda")) for _ in range(slots)]
            tl.key = key
        ev_in = [torch.cuda.Event() for _ in range(slots)]
        ev_comp = [torch.cuda.Event() for _ in range(slots)]
        ev_out = [None] * slots
        start = torch.cuda.Event()
        start.record(cur)
        for s in (s_in, s_comp, s_out):
            s.wait_event(start)
        for i, lo in enumerate(range(0, batch, step)):
            hi = min(batch, lo + step)
            m = hi - lo
            k = i % slots
            ctp_d, ptp_d, ct_d, pt_d, out_d, outp_d = tl.buf[k]
            if ev_out[k] is not None:
                s_in.wait_event(ev_out[k])
            with torch.cuda.stream(s_in):
                ctp_d[:m * per_ct].copy_(ctp_h[lo * per_ct:hi * per_ct], non_blocking=True)
                ptp_d[:m * per_pt].copy_(ptp_h[lo * per_pt:hi * per_pt], non_blocking=True)
            ev_in[k].record(s_in)
            s_comp.wait_event(ev_in[k])
            with torch.cuda.stream(s_comp):
                self.unpack_bits(ctp_d, qb, (m, 2, L, n), ct_d.dtype, out=ct_d[:m])
                self.unpack_bits(ptp_d, tb, (m, n), torch.int64, out=pt_d[:m])
                self.cpmul(ct_d[:m], pt_d[:m], out=out_d[:m])
                self.pack_bits(out_d[:m], qb, out=outp_d[:m * per_ct])
            ev_comp[k].record(s_comp)
            s_out.wait_event(ev_comp[k])
            with torch.cuda.stream(s_out):
                outp_h[lo * per_ct:hi * per_ct].copy_(outp_d[:m * per_ct], non_blocking=True)
            ev_out[k] = torch.cuda.Event()
            ev_out[k].record(s_out)
        cur.wait_stream(s_out)

    def pp_mul(self, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
        na = self._check_plain(a, "pp_mul")
        if b.shape != a.shape:
            raise ValueError("pp_mul: shape mismatch")
        out = torch.empty_like(a)
        check(self._lib.ctb_pp_mul(self._h, _ptr(a), _ptr(b), _ptr(out), na, _stream()), "ctb_pp_mul")
        return out
