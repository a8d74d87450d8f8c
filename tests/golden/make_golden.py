"""Generate golden vectors by running the REAL reference (not shipped, not run on the GPU box).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.json: SHA-256 digests (of canonical little-endian
uint64 residue arrays) plus a few leading values of reference outputs on
seeded inputs.  Inputs are re-drawn by the oracle with the same numpy calls in
the same order (same interpreter/numpy in this image), so one digest pins both
the oracle's sampling and its arithmetic.  The reference itself is only needed
here, never at test time.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from privtrain import he, linprot, packing, ring, transport  # noqa: E402
from privtrain.ring import RingElem, RingParams  # noqa: E402


def digest(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(arr, dtype=np.uint64), dtype="<u8").tobytes()).hexdigest()


def residues(elem: RingElem, primes) -> np.ndarray:
    return np.array([[int(c) % p for c in elem.coeffs] for p in primes], dtype=np.uint64)


def ct_residues(ct, primes) -> np.ndarray:
    return np.stack([residues(part, primes) for part in ct.parts])


def plain_vals(elem: RingElem) -> np.ndarray:
    return np.array([int(c) for c in elem.coeffs], dtype=np.uint64)


def protocol_case(params, job, keygen_seed=3, offline_seed=2, online_seed=4, timeout=60.0):
    cli, srv = he.He(params, he.BACKEND_RLWE), he.He(params, he.BACKEND_RLWE)
    keys = cli.keygen(keygen_seed)
    cpool, spool = linprot.TriplePool(), linprot.TriplePool()

    def client(end):
        linprot.setup_client(end, cli, keys)
        linprot.precompute_offline_client(end, cli, keys, np.random.default_rng(offline_seed), job.shape, 1, cpool)
        return linprot.precompute_online_client(end, cli, keys, np.random.default_rng(online_seed), job, cpool)

    def server(end):
        pks = linprot.setup_server(end, srv)
        linprot.precompute_offline_server(end, srv, pks, spool)
        linprot.precompute_online_server(end, srv, pks, spool)

    ce, se = transport.inproc_pair(capture=True, timeout=timeout)
    res, _ = transport.run_pair(client, server, ce, se)
    tr = ce.stats.transcript
    signed = np.asarray(packing.to_signed_matrix(np.asarray(res.tensor), params.t), dtype=np.int64)
    return {"c2s": hashlib.sha256(bytes(tr[transport.CLIENT])).hexdigest(),
            "s2c": hashlib.sha256(bytes(tr[transport.SERVER])).hexdigest(),
            "c2s_len": len(tr[transport.CLIENT]), "s2c_len": len(tr[transport.SERVER]),
            "tensor": digest(signed.astype(np.uint64)), "tensor_shape": list(signed.shape),
            "server_counts": srv.meter.snapshot()["counts"]}



def main():
    out: dict = {}
    # ------------------------------------------------------------ parameters
    P = he.default_he_params(4096)
    qp = list(P.cipher_ring.primes)
    tp = list(P.plain_ring.primes)
    out["p4096"] = {
        "q_primes": qp, "t_primes": tp,
        "psi": [ring._find_root_of_unity(8192, q) for q in qp],
        "delta_mod_q": [P.delta % q for q in qp],
        "relin_digits": P.relin_digits, "fresh_noise": P.fresh_noise,
        "noise_budget_bits": P.noise_budget.bit_length(),
        "aux_primes_15": ring.ntt_primes(4096, 30, 15),
    }
    plain_s = he.default_plain_params(512, prime_bits=17, primes=2)
    Ps = he.HeParams(he.default_cipher_params(512, plain_s.modulus), plain_s)
    out["p512"] = {"q_primes": list(Ps.cipher_ring.primes), "t_primes": list(Ps.plain_ring.primes)}
    out["p8192"] = {"q_primes": ring.ntt_primes(8192, 50, 3), "t_primes": ring.ntt_primes(8192, 18, 2),
                    "psi": [ring._find_root_of_unity(16384, q) for q in ring.ntt_primes(8192, 50, 3)]}

    # ------------------------------------------------------------ NTT per limb (ring.ntt_forward)
    ntt = []
    for i, q in enumerate(qp + out["p8192"]["q_primes"]):
        n = 4096 if i < len(qp) else 8192
        Rq = RingParams(n, q)
        a = RingElem.random(Rq, np.random.default_rng(100 + i))
        fa = ring.ntt_forward(a)
        back = ring.ntt_inverse(fa)
        assert back == a
        ntt.append({"n": n, "p": q, "seed": 100 + i, "in": digest(plain_vals(a)),
                    "fwd": digest(plain_vals(fa)), "fwd_head": [int(c) for c in fa.coeffs[:4]]})
    out["ntt"] = ntt

    # ------------------------------------------------------------ config 1: single CPMul, P4096
    ev = he.He(P, he.BACKEND_RLWE)
    keys = ev.keygen(1)
    rng = np.random.default_rng(1234)
    c0 = RingElem.random(P.cipher_ring, rng)
    c1 = RingElem.random(P.cipher_ring, rng)
    pt = RingElem.random(P.plain_ring, rng)
    ct = he.Ciphertext([c0, c1], P.fresh_noise, he.BACKEND_RLWE)
    prod = ev.cp_mul(ct, pt)
    m = RingElem.random(P.plain_ring, rng)
    cte = ev.encrypt(m, keys, rng)
    prode = ev.cp_mul(cte, pt)
    dec = ev.decrypt(prode, keys)
    assert dec == ring.ring_mul(m, pt)
    out["cfg1"] = {
        "keygen_seed": 1, "rng_seed": 1234,
        "sk": digest(np.array(keys.secret.to_signed(), dtype=np.int64).astype(np.uint64)),
        "pk0": digest(residues(keys.public[0], qp)), "pk1": digest(residues(keys.public[1], qp)),
        "relin0_b": digest(residues(keys.relin[0][0], qp)),
        "relin13_a": digest(residues(keys.relin[-1][1], qp)),
        "c_in": digest(ct_residues(ct, qp)), "pt": digest(plain_vals(pt)),
        "cpmul": digest(ct_residues(prod, qp)),
        "m": digest(plain_vals(m)), "enc": digest(ct_residues(cte, qp)),
        "enc_cpmul": digest(ct_residues(prode, qp)), "dec": digest(plain_vals(dec)),
        "dec_head": [int(c) for c in dec.coeffs[:4]],
        "cpmul_noise": prod.noise_estimate,
    }
    pa = RingElem.random(P.plain_ring, np.random.default_rng(55))
    pb = RingElem.random(P.plain_ring, np.random.default_rng(56))
    out["ppmul"] = {"seeds": [55, 56], "out": digest(plain_vals(ev.pp_mul(pa, pb)))}

    # ------------------------------------------------------------ CCMul + relin at N=512 (he_small)
    evs = he.He(Ps, he.BACKEND_RLWE)
    ks = evs.keygen(7)
    rng = np.random.default_rng(77)
    ma = RingElem.random(Ps.plain_ring, rng)
    mb = RingElem.random(Ps.plain_ring, rng)
    ca = evs.encrypt(ma, ks, rng)
    cb = evs.encrypt(mb, ks, rng)
    raw = evs.cc_mul_raw(ca, cb)
    rel = evs.relinearize(raw, ks)
    d = evs.decrypt(rel, ks)
    assert d == ring.ring_mul(ma, mb)
    qs = list(Ps.cipher_ring.primes)
    out["ccmul512"] = {
        "keygen_seed": 7, "rng_seed": 77,
        "ca": digest(ct_residues(ca, qs)), "cb": digest(ct_residues(cb, qs)),
        "raw": digest(ct_residues(raw, qs)), "relin": digest(ct_residues(rel, qs)),
        "dec": digest(plain_vals(d)), "raw_noise": raw.noise_estimate, "relin_noise": rel.noise_estimate,
    }
    # ------------------------------------------------------------ CCMul at N=4096 default params
    rng = np.random.default_rng(4242)
    ma = RingElem.random(P.plain_ring, rng)
    mb = RingElem.random(P.plain_ring, rng)
    ca = ev.encrypt(ma, keys, rng)
    cb = ev.encrypt(mb, keys, rng)
    raw = ev.cc_mul_raw(ca, cb)
    rel = ev.relinearize(raw, keys)
    out["ccmul4096"] = {"keygen_seed": 1, "rng_seed": 4242,
                        "ca": digest(ct_residues(ca, qp)), "raw": digest(ct_residues(raw, qp)),
                        "relin": digest(ct_residues(rel, qp)),
                        "dec": digest(plain_vals(ev.decrypt(rel, keys)))}

    # ------------------------------------------------------------ serialization (ring_to_bytes)
    blob = ring.ring_to_bytes(c0)
    out["serial"] = {"c0_bytes": hashlib.sha256(blob).hexdigest(), "len": len(blob),
                     "ct_bytes": hashlib.sha256(ev.ct_to_bytes(ct)).hexdigest()}

    # ------------------------------------------------------------ packing known answers
    out["packing"] = {
        "choose_tiles_64_64_5_4_4096": list(packing.choose_tiles(packing.ConvShape(64, 64, 5, 4), 4096)),
        "cfg3_plan": packing.plan_correlated(packing.ConvShape(28, 28, 5, 0), 4096).row_stride,
        "cfg4_plan": packing.plan_correlated(packing.ConvShape(32, 32, 3, 1), 4096).row_stride,
        "cfg4_gw_plan": [packing.plan_correlated(packing.ConvShape(32, 32, 32, 1), 4096).row_stride,
                         packing.plan_correlated(packing.ConvShape(32, 32, 32, 1), 4096).num_tiles],
    }
    # ------------------------------------------------------------ linprot sites
    js = linprot.conv_job("f", np.zeros((3, 32, 32), dtype=np.int64), np.zeros((64, 3, 3, 3), dtype=np.int64),
                          packing.ConvShape(32, 32, 3, 1), P.plain_ring).shape
    out["jobs"] = {"cfg4_fwd": [js.n_x, js.n_w, js.n_out, len(js.sites)],
                   "cfg4_fwd_sites_digest": hashlib.sha256(json.dumps(js.sites).encode()).hexdigest()}

    # ------------------------------------------------------------ two-party precompute protocol transcripts
    rng = np.random.default_rng(21)
    x = rng.integers(-40, 40, size=(2, 8, 8))
    w = rng.integers(-9, 9, size=(2, 2, 3, 3))
    proto = {"small_conv": {"x": x.tolist(), "w": w.tolist(),
                            **protocol_case(Ps, linprot.conv_job("c", x, w, packing.ConvShape(8, 8, 3, 1), Ps.plain_ring))}}
    rng = np.random.default_rng(22)
    x = rng.integers(-30, 30, size=(2, 6, 6))
    gy = rng.integers(-5, 5, size=(3, 4, 4))
    proto["small_gradw"] = {"x": x.tolist(), "gy": gy.tolist(),
                            **protocol_case(Ps, linprot.conv_grad_w_job("g", x, gy, packing.ConvShape(6, 6, 4, 1), Ps.plain_ring))}
    rng = np.random.default_rng(23)
    xf = rng.integers(-30, 30, size=40)
    wf = rng.integers(-30, 30, size=(5, 40))
    proto["small_fc"] = {"x": xf.tolist(), "w": wf.tolist(), **protocol_case(Ps, linprot.fc_job("fc", xf, wf, Ps.plain_ring))}
    rng = np.random.default_rng(3)
    x = rng.integers(0, 256, size=(1, 28, 28))
    w = rng.integers(-128, 128, size=(5, 1, 5, 5))
    proto["cfg3_image"] = {"x_seed": 3, **protocol_case(P, linprot.conv_job("cfg3", x, w, packing.ConvShape(28, 28, 5, 0), P.plain_ring))}
    out["protocol"] = proto

    path = Path(__file__).with_name("golden.json")
    path.write_text(json.dumps(out, indent=1, sort_keys=True))
    print("wrote", path)


if __name__ == "__main__":
    main()
