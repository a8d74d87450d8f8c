"""GPU parity of the drop-in he/ring mirror against the reference (golden digests)
and the oracle restatement.  Keys, ciphertexts, products and decryptions are
compared as exact residues."""
import hashlib

import numpy as np
import pytest

from _util import digest
from conftest import has_gpu
from oracle import he_ref as H
from oracle import ring_ref as R

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def res(elem):
    return elem.data.cpu().numpy().astype(np.uint64)


def ctres(ct):
    return ct.data.cpu().numpy().astype(np.uint64)


@pytest.fixture(scope="module")
def p4096():
    from paper_2409_16675_b200 import he
    return he.default_he_params(4096)


@pytest.fixture(scope="module")
def ev4096(p4096):
    from paper_2409_16675_b200 import he
    return he.He(p4096, he.BACKEND_RLWE)


@pytest.fixture(scope="module")
def keys4096(ev4096):
    return ev4096.keygen(1)


def test_params_mirror_reference(golden, p4096):
    assert list(p4096.cipher_ring.primes) == golden["p4096"]["q_primes"]
    assert list(p4096.plain_ring.primes) == golden["p4096"]["t_primes"]
    assert p4096.relin_digits == 14 and p4096.fresh_noise == golden["p4096"]["fresh_noise"]


def test_keygen_matches_reference(golden, keys4096):
    g = golden["cfg1"]
    s = np.array(keys4096.secret.to_signed(), dtype=np.int64).astype(np.uint64)
    assert digest(s) == g["sk"]
    assert digest(res(keys4096.public[0])) == g["pk0"]
    assert digest(res(keys4096.public[1])) == g["pk1"]
    assert digest(res(keys4096.relin[0][0])) == g["relin0_b"]
    assert digest(res(keys4096.relin[-1][1])) == g["relin13_a"]


def test_cfg1_encrypt_cpmul_decrypt(golden, p4096, ev4096, keys4096):
    from paper_2409_16675_b200 import he
    from paper_2409_16675_b200.ring import RingElem
    g = golden["cfg1"]
    rng = np.random.default_rng(g["rng_seed"])
    c0 = RingElem.random(p4096.cipher_ring, rng)
    c1 = RingElem.random(p4096.cipher_ring, rng)
    pt = RingElem.random(p4096.plain_ring, rng)
    ct = he.Ciphertext([c0, c1], p4096.fresh_noise, he.BACKEND_RLWE)
    assert digest(ctres(ct)) == g["c_in"] and digest(pt.coeffs) == g["pt"]
    prod = ev4096.cp_mul(ct, pt)
    assert digest(ctres(prod)) == g["cpmul"]
    assert prod.noise_estimate == g["cpmul_noise"]
    m = RingElem.random(p4096.plain_ring, rng)
    cte = ev4096.encrypt(m, keys4096, rng)
    assert digest(ctres(cte)) == g["enc"]
    prode = ev4096.cp_mul(cte, pt)
    assert digest(ctres(prode)) == g["enc_cpmul"]
    dec = ev4096.decrypt(prode, keys4096)
    assert digest(dec.coeffs) == g["dec"]
    assert [int(v) for v in dec.coeffs[:4]] == g["dec_head"]
    assert ev4096.meter.count("CPMul") >= 2 and ev4096.meter.count("Enc") >= 1


def test_serialization_matches_reference(golden, p4096, ev4096):
    from paper_2409_16675_b200 import he, ring
    from paper_2409_16675_b200.ring import RingElem
    rng = np.random.default_rng(1234)
    c0 = RingElem.random(p4096.cipher_ring, rng)
    c1 = RingElem.random(p4096.cipher_ring, rng)
    blob = ring.ring_to_bytes(c0)
    assert hashlib.sha256(blob).hexdigest() == golden["serial"]["c0_bytes"]
    back = ring.ring_from_bytes(blob, p4096.cipher_ring)
    assert back == c0
    ct = he.Ciphertext([c0, c1], p4096.fresh_noise, he.BACKEND_RLWE)
    assert hashlib.sha256(ev4096.ct_to_bytes(ct)).hexdigest() == golden["serial"]["ct_bytes"]
    ct2 = ev4096.ct_from_bytes(ev4096.ct_to_bytes(ct))
    assert np.array_equal(ctres(ct2), ctres(ct))
    # coefficient view equals the oracle's big integers
    want = R.sample_uniform(p4096.q, p4096.n, np.random.default_rng(1234))
    assert [int(v) for v in c0.coeffs[:16]] == [int(v) for v in want[:16]]


def test_ccmul_512_matches_reference(golden):
    from paper_2409_16675_b200 import he
    from paper_2409_16675_b200.ring import RingElem
    P = he.HeParams(he.default_cipher_params(512, he.default_plain_params(512, 17, 2).modulus),
                    he.default_plain_params(512, 17, 2))
    ev = he.He(P, he.BACKEND_RLWE)
    g = golden["ccmul512"]
    ks = ev.keygen(g["keygen_seed"])
    rng = np.random.default_rng(g["rng_seed"])
    ma = RingElem.random(P.plain_ring, rng)
    mb = RingElem.random(P.plain_ring, rng)
    ca = ev.encrypt(ma, ks, rng)
    cb = ev.encrypt(mb, ks, rng)
    assert digest(ctres(ca)) == g["ca"] and digest(ctres(cb)) == g["cb"]
    raw = ev.cc_mul_raw(ca, cb)
    assert digest(ctres(raw)) == g["raw"]
    assert raw.noise_estimate == g["raw_noise"]
    rel = ev.relinearize(raw, ks)
    assert digest(ctres(rel)) == g["relin"]
    assert rel.noise_estimate == g["relin_noise"]
    d = ev.decrypt(rel, ks)
    assert digest(d.coeffs) == g["dec"]
    # 3-part decrypt equals relinearised decrypt
    assert digest(ev.decrypt(raw, ks).coeffs) == g["dec"]
    assert ev.meter.count("Relin") == 1


def test_ccmul_4096_matches_reference(golden, p4096, ev4096, keys4096):
    from paper_2409_16675_b200.ring import RingElem
    g = golden["ccmul4096"]
    rng = np.random.default_rng(g["rng_seed"])
    ma = RingElem.random(p4096.plain_ring, rng)
    mb = RingElem.random(p4096.plain_ring, rng)
    ca = ev4096.encrypt(ma, keys4096, rng)
    cb = ev4096.encrypt(mb, keys4096, rng)
    assert digest(ctres(ca)) == g["ca"]
    raw = ev4096.cc_mul_raw(ca, cb)
    assert digest(ctres(raw)) == g["raw"]
    rel = ev4096.relinearize(raw, keys4096)
    assert digest(ctres(rel)) == g["relin"]
    assert digest(ev4096.decrypt(rel, keys4096).coeffs) == g["dec"]


def test_p8192_ccmul_cpmul_match_restatement():
    """N=8192, q = 3 x 50-bit: not expressible by the reference's he.He; checked
    against the oracle restatement (per-limb ring products + exact CRT rounding)."""
    from paper_2409_16675_b200 import he
    P = he.p8192_he_params()
    ev = he.He(P, he.BACKEND_RLWE)
    keys = ev.keygen(5)
    PR = H.p8192_params()
    okeys = H.keygen(PR, 5)
    assert np.array_equal(res(keys.public[0]), okeys["pk"][0])
    assert np.array_equal(res(keys.relin[3][0]), okeys["relin"][3][0])
    from paper_2409_16675_b200.ring import RingElem
    rng = np.random.default_rng(6)
    orng = np.random.default_rng(6)
    ma = RingElem.random(P.plain_ring, rng)
    mb = RingElem.random(P.plain_ring, rng)
    oma = R.sample_uniform(PR.t, PR.n, orng)
    omb = R.sample_uniform(PR.t, PR.n, orng)
    ca = ev.encrypt(ma, keys, rng)
    cb = ev.encrypt(mb, keys, rng)
    oca = H.encrypt(PR, oma, okeys["pk"], orng)
    ocb = H.encrypt(PR, omb, okeys["pk"], orng)
    assert np.array_equal(ctres(ca), oca) and np.array_equal(ctres(cb), ocb)
    raw = ev.cc_mul_raw(ca, cb)
    oraw = H.cc_mul_raw(PR, oca, ocb)
    assert np.array_equal(ctres(raw), oraw)
    rel = ev.relinearize(raw, keys)
    assert np.array_equal(ctres(rel), H.relinearize(PR, oraw, okeys["relin"]))
    dec = ev.decrypt(rel, keys)
    assert np.array_equal(dec.coeffs, H.pp_mul(PR, oma, omb))
    cp = ev.cp_mul(ca, mb)
    assert np.array_equal(ctres(cp), H.cp_mul(PR, oca, omb))


def test_errors_and_contracts(p4096, ev4096, keys4096):
    from paper_2409_16675_b200 import he
    from paper_2409_16675_b200.ring import RingElem
    rng = np.random.default_rng(3)
    a = ev4096.encrypt(RingElem.random(p4096.plain_ring, rng), keys4096, rng)
    b = ev4096.encrypt(RingElem.random(p4096.plain_ring, rng), keys4096, rng)
    raw = ev4096.cc_mul_raw(a, b)
    assert raw.nparts == 3
    with pytest.raises(he.PartCountError):
        ev4096.cp_mul(raw, RingElem.zeros(p4096.plain_ring))
    with pytest.raises(he.PartCountError):
        ev4096.cc_add(raw, a)
    with pytest.raises(he.PartCountError):
        ev4096.cc_mul(raw, a, keys4096)
    prod = ev4096.cc_mul(a, b, keys4096)
    deep = ev4096.cc_mul(prod, a, keys4096)
    with pytest.raises(he.NoiseOverflowError):
        ev4096.decrypt(deep, keys4096)
    with pytest.raises(ValueError):
        he.He(p4096, "bogus")
    # 3*5 = 15 (reference tests/test_he.py:78-87)
    three = ev4096.encrypt(RingElem.monomial(p4096.plain_ring, 3, 0), keys4096, rng)
    five = ev4096.encrypt(RingElem.monomial(p4096.plain_ring, 5, 0), keys4096, rng)
    out = ev4096.decrypt(ev4096.cc_mul(three, five, keys4096), keys4096).to_ints()
    assert out[0] == 15 and not any(out[1:])


def test_batched_apis_match_single_calls(p4096, ev4096, keys4096):
    from paper_2409_16675_b200 import he
    from paper_2409_16675_b200.ring import RingElem
    rng = np.random.default_rng(11)
    ms = [RingElem.random(p4096.plain_ring, rng) for _ in range(5)]
    pts = [RingElem.random(p4096.plain_ring, rng) for _ in range(5)]
    r1 = np.random.default_rng(12)
    batch = ev4096.encrypt_many(ms, keys4096, r1)
    r2 = np.random.default_rng(12)
    singles = [ev4096.encrypt(m, keys4096, r2) for m in ms]
    for i in range(5):
        assert np.array_equal(ctres(batch[i]), ctres(singles[i]))
    prod = ev4096.cp_mul_many(batch, pts)
    for i in range(5):
        assert np.array_equal(ctres(prod[i]), ctres(ev4096.cp_mul(singles[i], pts[i])))
    decs = ev4096.decrypt_many(prod, keys4096)
    from paper_2409_16675_b200 import ring
    for i in range(5):
        assert decs[i] == ring.ring_mul(ms[i], pts[i])


def test_device_sampler_distribution():
    """ctb_sample_draws: ternary u uniform on {-1,0,1}; e = clip(rint(N(0, sigma^2)), +-bound) (he.py:292-303)."""
    import torch
    from paper_2409_16675_b200 import _lib
    from paper_2409_16675_b200.device import RnsContext, _ptr, _stream
    from paper_2409_16675_b200.params import default_he_params
    P = default_he_params(4096)
    ctx = RnsContext.get(P.n, P.cipher_ring.primes, P.plain_ring.primes)
    B = 256

    def draw(seed, first):
        out = torch.empty((B, 3, P.n), dtype=torch.int8, device="cuda")
        _lib.check(ctx._lib.ctb_sample_draws(ctx._h, seed, first, P.noise_stddev, P.error_bound, _ptr(out), B,
                                             _stream()), "ctb_sample_draws")
        return out.to(torch.int64)

    d = draw(7, 0)
    u, e = d[:, 0].flatten(), d[:, 1:].flatten().double()
    for v in (-1, 0, 1):
        assert abs((u == v).double().mean().item() - 1 / 3) < 0.005
    assert u.abs().max().item() == 1
    assert abs(e.mean().item()) < 0.02
    assert abs(e.var().item() - (P.noise_stddev ** 2 + 1 / 12)) < 0.1
    assert e.abs().max().item() <= P.error_bound
    assert torch.equal(draw(7, 0), d)
    assert torch.equal(draw(7, 5)[:B - 5], d[5:])          # counter = global poly index
    assert not torch.equal(draw(8, 0), d)
    e1, e2 = d[:, 1].flatten().double(), d[:, 2].flatten().double()
    assert abs(torch.corrcoef(torch.stack([e1, e2]))[0, 1].item()) < 0.01
