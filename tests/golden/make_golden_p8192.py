"""Golden transcripts at the BASELINE N=8192 / 3 x 50-bit parameters (cfg2b / cfg5), produced by the
oracle's protocol restatement (oracle/linprot_ref.py) -- the reference cannot construct these
parameters (RingParams caps primes below 2^31, ring.py:134).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_p8192.py

Before writing, every 50-bit limb product the restatement uses is spot-checked against the REAL
reference's own per-limb ring product (`ring.ring_mul` on `RingParams(8192, q_i)`, the object-dtype
NTT path, ring.py:422-425) on random operands, and the restatement itself is pinned at N=512 / N=4096
to the reference's transcripts (tests/test_oracle.py).  Writes tests/golden/golden_p8192.json.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from oracle import he_ref as H  # noqa: E402
from oracle import linprot_ref as LP  # noqa: E402
from oracle import packing_ref as PR  # noqa: E402
from oracle import ring_ref as R  # noqa: E402


def digest(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(arr, dtype=np.uint64), dtype="<u8").tobytes()).hexdigest()


def spot_check_limbs(p):
    from privtrain import ring
    rng = np.random.default_rng(808)
    for q in p.q_primes:
        Rq = ring.RingParams(8192, q)
        a = ring.RingElem.random(Rq, rng)
        b = ring.RingElem.random(Rq, rng)
        want = np.array([int(c) for c in ring.ring_mul(a, b).coeffs], dtype=np.uint64)
        got = R.negacyclic_mul_mod(np.array([int(c) for c in a.coeffs], dtype=object),
                                   np.array([int(c) for c in b.coeffs], dtype=object), q)
        assert np.array_equal(np.asarray(got, dtype=np.uint64), want), q


def jobs(p):
    rng = np.random.default_rng(88)
    x = rng.integers(0, 256, size=(2, 8, 8))
    w = rng.integers(-128, 128, size=(3, 2, 3, 3))
    xg = rng.integers(0, 256, size=(2, 6, 6))
    gy = rng.integers(-128, 128, size=(3, 4, 4))
    xf = rng.integers(0, 256, size=40)
    wf = rng.integers(-128, 128, size=(5, 40))
    return {
        "conv": ({"x": x.tolist(), "w": w.tolist()}, PR.conv_job(x, w, 8, 8, 3, 1, p.n, p.t)),
        "gradw": ({"x": xg.tolist(), "gy": gy.tolist()}, PR.conv_grad_w_job(xg, gy, 6, 6, 4, 1, p.n, p.t)),
        "fc": ({"x": xf.tolist(), "w": wf.tolist()}, PR.fc_job(xf, wf, p.n, p.t)),
    }


def main():
    p = H.p8192_params()
    spot_check_limbs(p)
    out = {"params": {"n": p.n, "q_primes": list(p.q_primes), "t_primes": list(p.t_primes)}, "cases": {}}
    for name, (inputs, job) in jobs(p).items():
        res = LP.run_protocol(p, name, job)
        signed = PR.centered(job["extract"](res["out"]), p.t)
        out["cases"][name] = {
            **inputs,
            "c2s": hashlib.sha256(res["c2s"]).hexdigest(), "s2c": hashlib.sha256(res["s2c"]).hexdigest(),
            "c2s_len": len(res["c2s"]), "s2c_len": len(res["s2c"]),
            "maskprod": digest(np.stack(res["maskprod"])), "c_slots": digest(np.stack(res["c_slots"])),
            "p_slots": digest(np.stack(res["p_slots"])),
            "tensor": digest(signed.astype(np.uint64)), "tensor_shape": list(signed.shape),
        }
        print(name, "done", flush=True)
    path = Path(__file__).with_name("golden_p8192.json")
    path.write_text(json.dumps(out, indent=1, sort_keys=True))
    print("wrote", path)


if __name__ == "__main__":
    main()
