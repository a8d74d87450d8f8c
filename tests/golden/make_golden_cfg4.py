"""Golden transcripts for ONE cfg4 image, produced by the REAL reference (not shipped, not run on
the GPU box).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_cfg4.py

BASELINE cfg4 (conv 3x32x32 -> 64 filters 3x3, pad 1, N=4096 default parameters) lowered the way
the reference trainer lowers a conv layer's forward and backward (train.py:478-494):

  fwd  conv_job(x, w, ConvShape(32, 32, 3, 1))                       (train.py:333-351)
  gw   conv_grad_w_job(x, gy, ConvShape(32, 32, 32, 1))               (train.py:484-485)
  gx   conv_job(gy, rot180(w)^T, ConvShape(32, 32, 3, 3 - 1 - 1))     (train.py:486-493)

each run through the two-party precompute protocol (offline CCMul masks + online CPMul step,
linprot.py:387-485) exactly as make_golden.protocol_case does.  Inputs: x in [0, 2^8), w and gy in
[-2^7, 2^7), all from numpy default_rng(4) in that order.  The three jobs run in parallel processes
(about 3-4 minutes each on one core).  Writes tests/golden/golden_cfg4.json.
"""
from __future__ import annotations

import json
import multiprocessing as mp
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parent))


def inputs():
    rng = np.random.default_rng(4)
    x = rng.integers(0, 256, size=(3, 32, 32))
    w = rng.integers(-128, 128, size=(64, 3, 3, 3))
    gy = rng.integers(-128, 128, size=(64, 32, 32))
    return x, w, gy


def job_for(name):
    from privtrain import he, linprot, packing
    P = he.default_he_params(4096)
    x, w, gy = inputs()
    if name == "fwd":
        return P, linprot.conv_job("cfg4_fwd", x, w, packing.ConvShape(32, 32, 3, 1), P.plain_ring)
    if name == "gw":
        return P, linprot.conv_grad_w_job("cfg4_gw", x, gy, packing.ConvShape(32, 32, 32, 1), P.plain_ring)
    wrot = np.flip(w, axis=(2, 3)).transpose(1, 0, 2, 3).copy()
    return P, linprot.conv_job("cfg4_gx", gy, wrot, packing.ConvShape(32, 32, 3, 1), P.plain_ring)


def run(name):
    import make_golden
    t0 = time.time()
    P, job = job_for(name)
    case = make_golden.protocol_case(P, job, timeout=3600.0)
    case["js"] = [job.shape.n_x, job.shape.n_w, job.shape.n_out, len(job.shape.sites)]
    case["ref_seconds"] = round(time.time() - t0, 1)
    return name, case


def main():
    with mp.get_context("fork").Pool(3) as pool:
        res = dict(pool.map(run, ["fwd", "gw", "gx"]))
    out = {"inputs": "numpy default_rng(4): x (3,32,32) in [0,256), w (64,3,3,3) and gy (64,32,32) in [-128,128)",
           "cases": res}
    path = Path(__file__).with_name("golden_cfg4.json")
    path.write_text(json.dumps(out, indent=1, sort_keys=True))
    print("wrote", path)


if __name__ == "__main__":
    main()
