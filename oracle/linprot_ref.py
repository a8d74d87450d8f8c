"""Oracle restatement of the reference's precompute protocol (linprot.py) -- TEST ONLY.

Follows /root/reference/pkg/src/privtrain/:
  JobShape.to_bytes                 linprot.py:60-76
  setup_client / public_keys_to_bytes  linprot.py:334-340, he.py:491-498
  precompute_offline_client         linprot.py:387-404  (r_x, r_w = RingElem.random(plain) draws, then
                                                         encrypt each r_x, then each r_w, one rng)
  precompute_offline_server         linprot.py:407-427  (per site cc_mul + relinearize, CCAdd into slots)
  precompute_online_client          linprot.py:430-452  (encrypt x polys then w polys; masked x - r_x,
                                                         w - r_w; decrypt(c) - p per slot)
  precompute_online_server          linprot.py:455-485  (per site cp_mul(x, mw) + cp_mul(w, mx),
                                                         pp_mul(mx, mw); slots += [r_x r_w])
  _accumulate                       linprot.py:343-344
  wire.encode_blobs                 wire.py:55-59
  transport frames                  transport.py:112-113 (<u8 phase id><u32 len> + payload)
  he.ct_to_bytes                    he.py:459-461

Every ring product is the per-limb restatement of oracle.he_ref (exact at 30- and 50-bit limbs), so
this also states the protocol at the BASELINE N=8192 / 3 x 50-bit parameters the reference itself
cannot construct (its RingParams caps primes below 2^31, ring.py:134).  At the reference's own
parameters it is pinned to the reference transcripts in tests/golden (tests/test_oracle.py).
"""
from __future__ import annotations

import struct

import numpy as np

from . import he_ref as H
from . import ring_ref as R

PHASES = ("setup", "offline", "online", "nonlinear")


def frame(phase: str, payload: bytes) -> bytes:
    return struct.pack("<BI", PHASES.index(phase), len(payload)) + payload


def encode_blobs(blobs) -> bytes:
    return struct.pack("<I", len(blobs)) + b"".join(struct.pack("<I", len(b)) + b for b in blobs)


def job_shape_bytes(job_id: str, n_x: int, n_w: int, n_out: int, sites) -> bytes:
    jid = job_id.encode()
    flat = [v for s in sites for v in s]
    return (struct.pack("<H3I", len(jid), n_x, n_w, n_out) + jid + struct.pack("<I", len(sites))
            + struct.pack(f"<{len(flat)}I", *flat))


def cipher_bytes(p, rns: np.ndarray) -> bytes:
    return R.ring_to_bytes(H.rns_to_ints(p, rns), p.n, p.q)


def ct_bytes(p, ct: np.ndarray) -> bytes:
    return struct.pack("<B", ct.shape[0]) + b"".join(cipher_bytes(p, part) for part in ct)


def plain_bytes(p, vals) -> bytes:
    return R.ring_to_bytes(np.asarray(vals, dtype=np.uint64), p.n, p.t)


def public_keys_bytes(p, keys) -> bytes:
    polys = [keys["pk"][0], keys["pk"][1]]
    for bi, ai in keys["relin"]:
        polys += [bi, ai]
    return struct.pack("<H", len(polys)) + b"".join(cipher_bytes(p, x) for x in polys)


def _add(p, a, b):
    return H._add(p, a, b)


def offline_server(p, rx: np.ndarray, rw: np.ndarray, sites, n_out: int, relin) -> list:
    """Per site CCMul([r_x], [r_w]) (relinearised per site), CCAdd into its slot."""
    slots = [None] * n_out
    for xi, wi, oi in sites:
        prod = H.cc_mul(p, rx[xi], rw[wi], relin)
        slots[oi] = prod if slots[oi] is None else _add(p, slots[oi], prod)
    return slots


def online_server(p, xs, ws, mx, mw, sites, n_out: int, maskprod):
    """Per site c1 = cp_mul(x, mw), c2 = cp_mul(w, mx), slot += c1 + c2, p_slot += pp_mul(mx, mw);
    then every slot += [r_x r_w]."""
    c_slots, p_slots = [None] * n_out, [None] * n_out
    for xi, wi, oi in sites:
        c = _add(p, H.cp_mul(p, xs[xi], mw[wi]), H.cp_mul(p, ws[wi], mx[xi]))
        c_slots[oi] = c if c_slots[oi] is None else _add(p, c_slots[oi], c)
        pp = H.pp_mul(p, mx[xi], mw[wi])
        p_slots[oi] = pp if p_slots[oi] is None else H.plain_add(p, p_slots[oi], pp)
    for oi in range(n_out):
        c_slots[oi] = _add(p, c_slots[oi], maskprod[oi])
    return c_slots, p_slots


def run_protocol(p, job_id: str, job: dict, keygen_seed=3, offline_seed=2, online_seed=4) -> dict:
    """Both parties of setup + one offline bundle + one online job, as the reference's
    run_pair(client, server) does (tests/golden/make_golden.protocol_case): returns the
    client->server and server->client transcripts, the server's output slots and the client's
    decrypted result polys [n_out, N] (mod t)."""
    n_x, n_w, n_out, sites = job["n_x"], job["n_w"], job["n_out"], job["sites"]
    js = job_shape_bytes(job_id, n_x, n_w, n_out, sites)
    keys = H.keygen(p, keygen_seed)
    c2s, s2c = bytearray(), bytearray()
    c2s += frame("setup", public_keys_bytes(p, keys))
    # offline (count = 1)
    c2s += frame("offline", encode_blobs([b"off", js, struct.pack("<I", 1)]))
    rng = np.random.default_rng(offline_seed)
    r_x = [R.sample_uniform(p.t, p.n, rng) for _ in range(n_x)]
    r_w = [R.sample_uniform(p.t, p.n, rng) for _ in range(n_w)]
    enc_r = [H.encrypt(p, r, keys["pk"], rng) for r in r_x + r_w]
    c2s += frame("offline", encode_blobs([ct_bytes(p, c) for c in enc_r]))
    maskprod = offline_server(p, enc_r[:n_x], enc_r[n_x:], sites, n_out, keys["relin"])
    s2c += frame("offline", b"done")
    # online
    rng = np.random.default_rng(online_seed)
    xs = [H.encrypt(p, m, keys["pk"], rng) for m in job["x"]]
    ws = [H.encrypt(p, m, keys["pk"], rng) for m in job["w"]]
    mx = [H.plain_sub(p, m, r) for m, r in zip(job["x"], r_x)]
    mw = [H.plain_sub(p, m, r) for m, r in zip(job["w"], r_w)]
    blobs = [b"pre", js] + [ct_bytes(p, c) for c in xs + ws] + [plain_bytes(p, v) for v in mx + mw]
    c2s += frame("online", encode_blobs(blobs))
    c_slots, p_slots = online_server(p, xs, ws, mx, mw, sites, n_out, maskprod)
    s2c += frame("online", encode_blobs([ct_bytes(p, c) for c in c_slots] + [plain_bytes(p, v) for v in p_slots]))
    out = np.stack([H.plain_sub(p, H.decrypt(p, c, keys["s"]), pv) for c, pv in zip(c_slots, p_slots)])
    return {"c2s": bytes(c2s), "s2c": bytes(s2c), "c_slots": c_slots, "p_slots": p_slots, "out": out,
            "maskprod": maskprod}
