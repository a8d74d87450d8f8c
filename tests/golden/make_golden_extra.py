"""Extra golden transcripts from the REAL reference (not shipped, not run on the GPU box):
protocol b -- direct CCMul on the server, CryptoTrain-B (linprot.py:352-379) -- on small jobs at
the N=512 test parameters, both directions of the two-party transcript.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_extra.py
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from privtrain import he, linprot, packing, transport  # noqa: E402


def digest(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(arr, dtype=np.uint64), dtype="<u8").tobytes()).hexdigest()


def protocol_b_case(params, job, keygen_seed=3, online_seed=4):
    cli, srv = he.He(params, he.BACKEND_RLWE), he.He(params, he.BACKEND_RLWE)
    keys = cli.keygen(keygen_seed)

    def client(end):
        linprot.setup_client(end, cli, keys)
        return linprot.linear_b_client(end, cli, keys, np.random.default_rng(online_seed), job)

    def server(end):
        pks = linprot.setup_server(end, srv)
        linprot.linear_b_server(end, srv, pks)

    ce, se = transport.inproc_pair(capture=True, timeout=600.0)
    res, _ = transport.run_pair(client, server, ce, se)
    tr = ce.stats.transcript
    signed = np.asarray(packing.to_signed_matrix(np.asarray(res.tensor), params.t), dtype=np.int64)
    return {"c2s": hashlib.sha256(bytes(tr[transport.CLIENT])).hexdigest(),
            "s2c": hashlib.sha256(bytes(tr[transport.SERVER])).hexdigest(),
            "c2s_len": len(tr[transport.CLIENT]), "s2c_len": len(tr[transport.SERVER]),
            "tensor": digest(signed.astype(np.uint64)), "tensor_shape": list(signed.shape),
            "server_counts": srv.meter.snapshot()["counts"]}


def main():
    plain = he.default_plain_params(512, prime_bits=17, primes=2)
    Ps = he.HeParams(he.default_cipher_params(512, plain.modulus), plain)
    rng = np.random.default_rng(61)
    x = rng.integers(-40, 40, size=(2, 8, 8))
    w = rng.integers(-9, 9, size=(2, 2, 3, 3))
    out = {"protocol_b": {
        "conv": {"x": x.tolist(), "w": w.tolist(),
                 **protocol_b_case(Ps, linprot.conv_job("bc", x, w, packing.ConvShape(8, 8, 3, 1), Ps.plain_ring))}}}
    xf = rng.integers(-30, 30, size=40)
    wf = rng.integers(-30, 30, size=(5, 40))
    out["protocol_b"]["fc"] = {"x": xf.tolist(), "w": wf.tolist(),
                               **protocol_b_case(Ps, linprot.fc_job("bf", xf, wf, Ps.plain_ring))}
    path = Path(__file__).with_name("golden_extra.json")
    path.write_text(json.dumps(out, indent=1, sort_keys=True))
    print("wrote", path)


if __name__ == "__main__":
    main()
