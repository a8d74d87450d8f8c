"""Trainer-facing engine over the device HE path (reference train.py:232-290, session.py:33-93).

`DeviceSecureEngine` exposes the reference `SecureEngine`'s primitives with the
same names, arguments, return values and errors, so the reference `Trainer`
(train.py:296-545) can drive the device path unchanged:

  conv_forward(x, w, shape, job_id)   -> conv_job        (train.py:263-266)
  conv_pairwise(x, gy, shape, job_id) -> conv_grad_w_job (train.py:268-271)
  fc(w, x, job_id)                    -> fc_job          (train.py:273-275)
  outer(g, x, job_id)                 -> outer_job       (train.py:277-279)
  affine(x, gamma, job_id)            -> affine_job      (train.py:281-283)
  relu(x), maxpool4(windows)          -> the OT protocol (train.py:285-297)

Outputs are the centred mod-t results checked against the 2*bits budget
(train.py:258-261), bit-identical to `PlainEngine` because the protocol is
exact ring arithmetic.  Both parties run co-resident on one GPU
(`DeviceSession`): client encryption, the server's fused online step
(`ctb_linear_online`) and client decryption exchange device buffers instead
of wire bytes; the byte-level two-party path is `linprot`'s channel functions.

The non-linear primitives are NOT computed here: `relu` / `maxpool4` hand the
values, as 2^bits residues (mpc.from_signed), to an injected non-linear protocol
with the signature of the reference's `SecureSession.nonlinear(op, values, bits)`
(session.py:78-84 -> mpc.client_nonlinear, the OT protocol of mpc.py), and map its
reconstruction back with mpc.to_signed -- exactly SecureEngine.relu / maxpool4
(train.py:278-290).  The OT protocol stays in the reference; an
engine without one refuses to run a non-linear layer.  `cleartext_nonlinear` is
an explicitly named TEST DOUBLE returning what the OT protocol reconstructs.

Beyond the reference (the trainer lowerings BASELINE configs 3 and 5 need,
SURVEY.md Appendix A): `conv_forward_strided` (stride-1 job + subsample) and
`fc_chunked` / `outer_chunked` (in_dim split into chunks of at most N).
"""
from __future__ import annotations

import collections
import time

import numpy as np
import torch

from . import linprot, packing, workloads
from .he import CiphertextBatch, HeParams
from .linprot import JobShape, LinearJob, PoolExhaustedError

PROTOCOL_B = "b"
PROTOCOL_PRECOMPUTE = "precompute"


class TrainError(Exception):
    """train.py:31-32."""


class FixedPointOverflowError(TrainError):
    """train.py:35-36."""


def check_range(arr: np.ndarray, bits: int) -> np.ndarray:
    """train.py:69-76: values must lie in [-2^(bits-1), 2^(bits-1))."""
    lim = 1 << (bits - 1)
    if arr.size and (arr.max(initial=0) >= lim or arr.min(initial=0) < -lim):
        raise FixedPointOverflowError(
            f"value magnitude {max(abs(int(arr.max(initial=0))), abs(int(arr.min(initial=0))))} "
            f"breaches the {bits}-bit budget")
    return arr


def _sync():
    torch.cuda.synchronize()


class DeviceSession:
    """Client + server of one session, co-resident on the GPU (session.py:33-119).

    `ensure_offline(shapes, count)` tops the pool up to `count` precomputed
    mask products per job shape (session.py:54-65); `linear(job)` runs one
    online job and returns the extracted mod-t tensor (session.py:67-76).
    Under protocol "b" every call runs per-site CCMul online instead.
    """

    def __init__(self, params: HeParams, protocol: str = PROTOCOL_PRECOMPUTE, seed: int = 0,
                 keygen_seed: int = 1, auto_offline: bool = False):
        if protocol not in (PROTOCOL_B, PROTOCOL_PRECOMPUTE):
            raise ValueError(f"unknown protocol {protocol!r}")
        self.params = params
        self.protocol = protocol
        self.auto_offline = auto_offline
        self.parties = workloads.Session.create(params, keygen_seed)
        self.gen = torch.Generator(device="cuda")
        self.gen.manual_seed(seed)
        self.mask_gen = torch.Generator(device="cuda")
        self.mask_gen.manual_seed(seed + 1)
        self._pool: dict[str, collections.deque] = collections.defaultdict(collections.deque)
        self.online_seconds = 0.0
        self.offline_seconds = 0.0
        self.jobs_run = 0

    @property
    def client(self):
        return self.parties.client

    @property
    def server(self):
        return self.parties.server

    def available(self, job_id: str) -> int:
        return len(self._pool[job_id])

    def ensure_offline(self, shapes: list[JobShape], count: int):
        if self.protocol != PROTOCOL_PRECOMPUTE:
            return
        t0 = time.perf_counter()
        self.server.meter.set_phase("offline")
        try:
            for js in shapes:
                for _ in range(count - self.available(js.job_id)):
                    self._add_bundle(js)
            _sync()
        finally:
            self.server.meter.set_phase("online")
        self.offline_seconds += time.perf_counter() - t0

    def _add_bundle(self, js: JobShape):
        dummy = LinearJob(js, torch.empty((js.n_x, 0), dtype=torch.int64),
                          torch.empty((js.n_w, 0), dtype=torch.int64))
        bundle, prod = workloads.offline(self.parties, dummy, self.mask_gen)
        self._pool[js.job_id].append((bundle, prod))

    def _take(self, js: JobShape):
        q = self._pool[js.job_id]
        if not q:
            if not self.auto_offline:
                raise PoolExhaustedError(f"no precomputed triples left for job {js.job_id!r}")
            self.ensure_offline([js], 1)
        bundle, prod = q.popleft()
        if (bundle.r_x.shape[0], bundle.r_w.shape[0], prod.data.shape[0]) != (js.n_x, js.n_w, js.n_out):
            raise linprot.LinProtError(f"pool entry for {js.job_id!r} has a different job shape")
        return bundle, prod

    def _online(self, job: LinearJob, decode: bool, centered: bool) -> torch.Tensor:
        t0 = time.perf_counter()
        if self.protocol == PROTOCOL_B:
            out = self._linear_b(job)
            if decode and job.extract is not None:
                out = job.extract(out)
                if centered:
                    out = packing.to_signed_tensor(out, self.params.t)
        else:
            bundle, prod = self._take(job.shape)
            out = workloads.online(self.parties, job, bundle, prod, self.gen, decode=decode, centered=centered)
        _sync()
        self.online_seconds += time.perf_counter() - t0
        self.jobs_run += 1
        return out

    def linear_polys(self, job: LinearJob) -> torch.Tensor:
        """[n_out, N] mod-t output polynomials of one job."""
        return self._online(job, decode=False, centered=False)

    def linear(self, job: LinearJob) -> torch.Tensor:
        """The job's extracted tensor, residues mod t (session.py:67-76 -> job.extract)."""
        if job.out is None:
            out = self.linear_polys(job)
            return job.extract(out) if job.extract else out
        return self._online(job, decode=True, centered=False)

    def linear_signed(self, job: LinearJob) -> torch.Tensor:
        """The job's extracted tensor centred into (-t/2, t/2] (to_signed_matrix), decoded in the
        decrypt epilogue."""
        if job.out is None:
            return packing.to_signed_tensor(self.linear(job), self.params.t)
        return self._online(job, decode=True, centered=True)

    def _linear_b(self, job: LinearJob) -> torch.Tensor:
        js, cli, srv = job.shape, self.client, self.server
        keys = self.parties.keys
        fresh = srv.params.fresh_noise
        cx, cw = job.encrypt_operands(cli, keys, self.gen)
        xs = CiphertextBatch(cx.data, fresh, cx.backend_tag, cx._cipher)
        ws = CiphertextBatch(cw.data, fresh, cw.backend_tag, cw._cipher)
        slots = linprot._sites_ccmul_sum(srv, self.parties.pks, xs, ws, js)
        return cli.decrypt_values(slots, keys)

    def report(self) -> dict:
        return {"server_meter": self.server.meter.snapshot(), "client_meter": self.client.meter.snapshot(),
                "online_seconds": self.online_seconds, "offline_seconds": self.offline_seconds,
                "jobs": self.jobs_run}


def _umod(arr, bits: int) -> np.ndarray:
    return np.asarray(arr, dtype=np.int64).astype(np.uint64) & np.uint64((1 << bits) - 1)


def from_signed(x, bits: int) -> np.ndarray:
    """mpc.from_signed (mpc.py:114-115): signed values -> residues mod 2^bits."""
    return _umod(x, bits)


def to_signed(x, bits: int) -> np.ndarray:
    """mpc.to_signed (mpc.py:108-111)."""
    v = (np.asarray(x, dtype=np.uint64) & np.uint64((1 << bits) - 1)).astype(np.int64)
    half = 1 << (bits - 1)
    return np.where(v >= half, v - (1 << bits), v)


def cleartext_nonlinear(op: str, values: np.ndarray, bits: int) -> np.ndarray:
    """TEST DOUBLE for the OT non-linear protocol: returns, in the clear, what mpc.client_nonlinear
    reconstructs (relu: max(x, 0); maxpool: the max over the 4 window rows), as 2^bits residues.
    Never use it where the secure protocol is required -- pass SecureSession.nonlinear instead."""
    x = to_signed(values, bits)
    if op == "relu":
        out = np.maximum(x, 0)
    elif op == "maxpool":
        out = x.max(axis=0)
    else:
        raise TrainError(f"unknown nonlinear op {op!r}")
    return from_signed(out, bits)


class DeviceSecureEngine:
    """SecureEngine-compatible primitives on the device path (train.py:232-290).

    `nonlinear(op, values, bits) -> values` is the secure non-linear protocol, e.g. the bound
    method `SecureSession.nonlinear` of a reference session (session.py:78-84), which runs the
    OT protocol of mpc.py against the reference server loop."""

    name = "secure"

    def __init__(self, session: DeviceSession, plain_ring=None, bits: int = 32,
                 scheme: str = packing.SCHEME_CORRELATED, nonlinear=None):
        self.session = session
        self.nonlinear = nonlinear
        self.ring = plain_ring if plain_ring is not None else session.params.plain_ring
        self.bits = bits
        self.scheme = scheme
        self.scheme_counts = {packing.SCHEME_CORRELATED: 0, packing.SCHEME_BASELINE: 0}
        if self.ring.modulus <= (1 << (bits + 1)):
            raise TrainError("plain modulus too small for the fixed-point budget")

    def _jid(self, stem: str) -> str:
        return stem

    def _signed(self, t: torch.Tensor) -> np.ndarray:
        signed = packing.to_signed_tensor(t, self.ring.modulus).cpu().numpy().astype(np.int64)
        return check_range(signed, 2 * self.bits)

    def _run(self, job: LinearJob) -> np.ndarray:
        # train.py:251-254: session.linear -> to_signed_matrix -> check_range; the centring runs
        # in the decrypt epilogue here
        return check_range(self.session.linear_signed(job).cpu().numpy().astype(np.int64), 2 * self.bits)

    # -- the reference primitives ----------------------------------------------------------

    def conv_forward(self, x, w, shape: packing.ConvShape, job_id: str = "conv") -> np.ndarray:
        self.scheme_counts[self.scheme] += 1
        return self._run(linprot.conv_job(self._jid(job_id), x, w, shape, self.ring, self.scheme))

    def conv_pairwise(self, x, gy, shape: packing.ConvShape, job_id: str = "convgw") -> np.ndarray:
        self.scheme_counts[packing.SCHEME_CORRELATED] += 1
        return self._run(linprot.conv_grad_w_job(self._jid(job_id), x, gy, shape, self.ring))

    def fc(self, w, x, job_id: str = "fc") -> np.ndarray:
        return self._run(linprot.fc_job(self._jid(job_id), x, w, self.ring))

    def outer(self, g, x, job_id: str = "outer") -> np.ndarray:
        return self._run(linprot.outer_job(self._jid(job_id), g, x, self.ring))

    def affine(self, x, gamma: int, job_id: str = "bn") -> np.ndarray:
        return self._run(linprot.affine_job(self._jid(job_id), x, int(gamma), self.ring))

    def _nl(self):
        if self.nonlinear is None:
            raise TrainError("no non-linear protocol attached: construct the engine with "
                             "nonlinear=SecureSession.nonlinear (the reference OT path, session.py:78-84)")
        return self.nonlinear

    def relu(self, x: np.ndarray) -> np.ndarray:
        """train.py:278-283: from_signed -> session.nonlinear("relu") -> to_signed."""
        x = np.asarray(x)
        flat = from_signed(x.ravel(), self.bits)
        out = self._nl()("relu", flat, self.bits)
        return to_signed(out, self.bits).reshape(x.shape)

    def maxpool4(self, windows: np.ndarray) -> np.ndarray:
        """train.py:285-290: the 4 window rows go to session.nonlinear("maxpool")."""
        vals = from_signed(np.asarray(windows), self.bits)
        out = self._nl()("maxpool", vals, self.bits)
        return to_signed(out, self.bits)

    # -- lowerings the BASELINE configs need (not in the reference) ----------------------

    def conv_forward_strided(self, x, w, shape: packing.ConvShape, stride: int,
                             job_id: str = "conv") -> np.ndarray:
        """Stride-s convolution as the stride-1 job subsampled (SPEC.md:544 lowering); the
        subsampling is the job's extraction map, so only the kept outputs are decrypted."""
        self.scheme_counts[self.scheme] += 1
        x = np.asarray(x) if not isinstance(x, torch.Tensor) else x
        xb = x[None] if x.ndim == 3 else x[None, None]
        return self._run(linprot.conv_job_batch(self._jid(job_id), xb, w, shape, self.ring, stride=stride))[0]

    def fc_chunked(self, w, x, job_id: str = "fc") -> np.ndarray:
        """y = W x for in_dim > N: one fc job per N-column chunk, summed client-side."""
        w, x = np.asarray(w, dtype=np.int64), np.asarray(x, dtype=np.int64).reshape(-1)
        n = self.ring.n
        if w.shape[1] <= n:
            return self.fc(w, x, job_id)
        acc = None
        for k, lo in enumerate(range(0, w.shape[1], n)):
            part = self.fc(w[:, lo:lo + n], x[lo:lo + n], f"{job_id}.k{k}")
            acc = part if acc is None else acc + part
        return check_range(acc, 2 * self.bits)

    def outer_chunked(self, g, x, job_id: str = "outer") -> np.ndarray:
        """g x^T for len(x) > N: column blocks of at most N."""
        g, x = np.asarray(g, dtype=np.int64).reshape(-1), np.asarray(x, dtype=np.int64).reshape(-1)
        n = self.ring.n
        if x.size <= n:
            return self.outer(g, x, job_id)
        return np.concatenate([self.outer(g, x[lo:lo + n], f"{job_id}.k{k}")
                               for k, lo in enumerate(range(0, x.size, n))], axis=1)

    # -- batched form (one library call per primitive for a whole minibatch) -------------

    def conv_forward_batch(self, xs, w, shape: packing.ConvShape, job_id: str = "conv") -> np.ndarray:
        """conv_forward for a batch of images [B, cin, H, W] in one fused job."""
        self.scheme_counts[self.scheme] += len(xs)
        return self._run(linprot.conv_job_batch(job_id, xs, w, shape, self.ring))

    def conv_pairwise_batch(self, xs, gys, shape: packing.ConvShape, job_id: str = "convgw") -> np.ndarray:
        self.scheme_counts[packing.SCHEME_CORRELATED] += len(xs)
        return self._run(linprot.conv_grad_w_job_batch(job_id, xs, gys, shape, self.ring))

    def batch_shape(self, jobs_or_shapes, job_id: str) -> JobShape:
        """The block-diagonal JobShape the *_batch primitives consume (for ensure_offline)."""
        shapes = [j.shape if isinstance(j, LinearJob) else j for j in jobs_or_shapes]
        sites, xo, wo, oo = [], 0, 0, 0
        for s in shapes:
            sites.extend((a + xo, b + wo, c + oo) for a, b, c in s.sites)
            xo, wo, oo = xo + s.n_x, wo + s.n_w, oo + s.n_out
        return JobShape(job_id, xo, wo, oo, tuple(sites))
