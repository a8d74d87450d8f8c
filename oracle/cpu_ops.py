"""CPU baseline for the protocol configs (cfg3/cfg4/cfg5) and cfg2b -- BENCH ONLY.

Times the reference's per-operation costs with the oracle restatement (oracle/he_ref.py: Enc
he.py:307-323, Dec :329-351, CPMul :366-382, CCAdd :355-364, PPMul :441-445, CCMul = cc_mul_raw +
relinearize :384-439) on every host core at once (one fork process per core, each on its own fresh
inputs, so memory-bandwidth contention between cores is included), and extrapolates a workload
from the operation counts the reference's meters record for it (linprot.py:387-485: online per job
Enc n_x + n_w, CPMul 2 S, CCAdd 2 S, PPMul S, Dec n_out; offline Enc n_x + n_w, CCMul S,
CCAdd S - n_out).  The reference itself is pure Python and runs its sites one after another, so the
all-core figure (work / cores) is generous to it.  `kind = "port"` in bench.py's JSON.
"""
from __future__ import annotations

import multiprocessing as mp
import time

import numpy as np

from . import he_ref as H
from . import ring_ref as R
from .cpu_baseline import usable_cores

OPS = ("Enc", "Dec", "CPMul", "CCAdd", "PPMul", "CCMul")
_STATE: dict = {}


def _params(name: str):
    return H.default_params(4096) if name == "p4096" else H.p8192_params()


def _setup(name: str, seed: int):
    P = _params(name)
    keys = H.keygen(P, 3 + seed)
    rng = np.random.default_rng(100 + seed)
    ms = [R.sample_uniform(P.t, P.n, rng) for _ in range(2)]
    cts = [H.encrypt(P, m, keys["pk"], rng) for m in ms]
    _STATE.update(name=name, P=P, keys=keys, rng=rng, ms=ms, cts=cts)


def _one(op: str):
    P, keys, rng, ms, cts = (_STATE[k] for k in ("P", "keys", "rng", "ms", "cts"))
    if op == "Enc":
        H.encrypt(P, R.sample_uniform(P.t, P.n, rng), keys["pk"], rng)
    elif op == "Dec":
        H.decrypt(P, cts[0], keys["s"])
    elif op == "CPMul":
        H.cp_mul(P, cts[0], R.sample_uniform(P.t, P.n, rng))
    elif op == "CCAdd":
        H._add(P, cts[0], cts[1])
    elif op == "PPMul":
        H.pp_mul(P, ms[0], R.sample_uniform(P.t, P.n, rng))
    elif op == "CCMul":
        H.cc_mul(P, cts[0], cts[1], keys["relin"])


def _worker(args):
    name, seed, reps = args
    if _STATE.get("name") != name:
        _setup(name, seed)
    out = {}
    for op, n in reps.items():
        t0 = time.perf_counter()
        for _ in range(n):
            _one(op)
        out[op] = (time.perf_counter() - t0) / max(n, 1)
    return out


def op_seconds(name: str, reps: dict, procs: int | None = None) -> tuple[dict, int, float]:
    """Mean single-operation seconds per op, measured with `procs` processes running concurrently
    (default: every usable core).  Returns (seconds per op, processes, wall seconds)."""
    procs = procs or usable_cores()
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_worker, [(name, s, reps) for s in range(procs)], chunksize=1)
    wall = time.perf_counter() - t0
    return {op: float(np.mean([r[op] for r in res])) for op in reps}, procs, wall


def job_counts(n_x: int, n_w: int, n_out: int, sites: int) -> dict:
    """The reference meters' operation counts of one job (client + server, both phases)."""
    return {
        "online": {"Enc": n_x + n_w, "CPMul": 2 * sites, "CCAdd": 2 * sites, "PPMul": sites, "Dec": n_out},
        "offline": {"Enc": n_x + n_w, "CCMul": sites, "CCAdd": max(sites - n_out, 0)},
    }


def extrapolate(counts: dict, secs: dict, cores: int) -> float:
    """Seconds for the counted operations spread perfectly over `cores` processes."""
    return sum(n * secs[op] for op, n in counts.items()) / cores
