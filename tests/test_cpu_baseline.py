"""The CPU-baseline legs of bench.py (the reference's CPU path, timed beside the GPU) compute what the
reference computes: the CPMul port reproduces the reference's cfg1 CPMul (golden digest from the real
reference), and the protocol extrapolation counts the operations the reference meters record for the
cfg4 jobs (golden server meter counts, tests/golden/golden_cfg4.json)."""
import json
from pathlib import Path

import numpy as np

from _util import digest
from oracle import cpu_baseline as CB
from oracle import cpu_ops
from oracle import he_ref as H
from oracle import ring_ref as R

GOLD = Path(__file__).resolve().parent / "golden"


def test_cpmul_port_matches_reference_cfg1(golden):
    """oracle/cpu_baseline.reference_cp_mul (the reference's object-dtype data path: residue
    extraction, per-prime NTT, CRT recombination) == He.cp_mul of the reference."""
    P = H.default_params(4096)
    g = golden["cfg1"]
    rng = np.random.default_rng(g["rng_seed"])
    c0 = R.sample_uniform(P.q, P.n, rng)
    c1 = R.sample_uniform(P.q, P.n, rng)
    pt = R.sample_uniform(P.t, P.n, rng)
    out = CB.reference_cp_mul([np.asarray(c0, dtype=object), np.asarray(c1, dtype=object)], pt, P)
    res = np.stack([H.ints_to_rns(P, part) for part in out])
    assert digest(res) == g["cpmul"]


def test_protocol_op_counts_match_reference_meters():
    cases = json.loads((GOLD / "golden_cfg4.json").read_text())["cases"]
    for name, case in cases.items():
        n_x, n_w, n_out, sites = case["js"]
        counts = cpu_ops.job_counts(n_x, n_w, n_out, sites)
        server = case["server_counts"]
        for phase in ("online", "offline"):
            for op in ("CPMul", "PPMul", "CCMul"):
                assert counts[phase].get(op, 0) == server.get(f"{phase}:{op}", 0), (name, phase, op)
        assert counts["online"]["CCAdd"] == server["online:CCAdd"]
        assert counts["offline"]["CCAdd"] == server.get("offline:CCAdd", 0)


def test_extrapolation_arithmetic():
    secs = {"Enc": 0.02, "CPMul": 0.03, "CCAdd": 0.001, "PPMul": 0.01, "Dec": 0.015}
    c = cpu_ops.job_counts(3, 192, 64, 192)["online"]
    want = (195 * 0.02 + 384 * 0.03 + 384 * 0.001 + 192 * 0.01 + 64 * 0.015) / 4
    assert abs(cpu_ops.extrapolate(c, secs, 4) - want) < 1e-12
