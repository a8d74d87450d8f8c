"""CPU baseline: the reference's CPMul data path, restated -- TEST/BENCH ONLY.

Times the same work He.cp_mul does per call in the reference
(he.py:366-382 -> _lift he.py:325-327 -> ring.ring_mul x2 ring.py:404 ->
_crt_ntt_mul ring.py:462-474 -> _fwd_residue ring.py:454-459 ->
_NttPlan.forward/inverse ring.py:186-217 -> _crt_combine ring.py:486-491):
ciphertext parts are object arrays of Python ints in [0, q), each of the L
primes extracts residues, runs the forward NTTs (the lifted plaintext's is
memoised across the two parts as RingElem._fwd_cache does), a
pointwise product and an inverse NTT, and the L residue vectors are
recombined into Python ints.  `kind = "port"` in bench.py's JSON.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from . import he_ref as H
from . import ring_ref as R


def _crt(residues, primes, q):
    acc = np.zeros(len(residues[0]), dtype=object)
    for r, p in zip(residues, primes):
        m = q // p
        acc += r.astype(object) * (m * pow(m, -1, p))
    return acc % q


def reference_cp_mul(parts_int, pt_u64, P: H.HeParamsRef):
    """One CPMul exactly along the reference's representation and call path."""
    q, t = P.q, P.t
    half = t // 2
    lifted = np.array([int(c) - t if int(c) > half else int(c) for c in pt_u64], dtype=object) % q
    out = []
    lifted_fwd = {}  # RingElem._fwd_cache of the lifted plaintext (ring.py:454-459)
    for part in parts_int:
        residues = []
        for p in P.q_primes:
            plan = R.NttPlan(P.n, p)
            fa = plan.forward((part % p).astype(np.uint64))
            if p not in lifted_fwd:
                lifted_fwd[p] = plan.forward((lifted % p).astype(np.uint64))
            residues.append(plan.inverse(fa * lifted_fwd[p] % np.uint64(p)))
        out.append(_crt(residues, P.q_primes, q))
    return out


def _make_inputs(P, seed, count):
    rng = np.random.default_rng(seed)
    cts = [[R.sample_uniform(P.q, P.n, rng) for _ in range(2)] for _ in range(count)]
    pts = [R.sample_uniform(P.t, P.n, rng) for _ in range(count)]
    return cts, pts


_STATE: dict = {}


def _worker(args):
    seed, n_ops, n = args
    if _STATE.get("n") != n:
        P = H.default_params(n)
        _STATE.update(n=n, P=P, inputs=_make_inputs(P, seed, 2))
        reference_cp_mul(_STATE["inputs"][0][0], _STATE["inputs"][1][0], P)  # warm twiddle plans
    P = _STATE["P"]
    cts, pts = _STATE["inputs"]
    t0 = time.perf_counter()
    for k in range(n_ops):
        reference_cp_mul(cts[k % 2], pts[k % 2], P)
    return n_ops, time.perf_counter() - t0


def usable_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class CpuPool:
    """Persistent fork pool; one independent ciphertext stream per process."""

    def __init__(self, procs: int | None = None, n: int = 4096):
        self.procs = procs or usable_cores()
        self.n = n
        self._pool = mp.get_context("fork").Pool(self.procs)
        # warm every worker's plan cache
        self._pool.map(_worker, [(s, 1, n) for s in range(self.procs)], chunksize=1)

    def run(self, ops_per_proc: int) -> tuple[int, float]:
        """Run ops_per_proc CPMuls in every process; return (ops, wall seconds)."""
        t0 = time.perf_counter()
        res = self._pool.map(_worker, [(1000 + s, ops_per_proc, self.n) for s in range(self.procs)], chunksize=1)
        wall = time.perf_counter() - t0
        self.last_per_op = max(r[1] / max(r[0], 1) for r in res)
        return sum(r[0] for r in res), wall

    def close(self):
        self._pool.terminate()
