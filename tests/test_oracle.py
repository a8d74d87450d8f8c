"""The CPU oracle (oracle/) pinned against the reference's own outputs (golden.json)
and the reference tests' known answers.  No GPU needed."""
import numpy as np
import pytest

from _util import digest
from oracle import he_ref as H
from oracle import ring_ref as R


def test_params_match_reference(golden):
    P = H.default_params(4096)
    g = golden["p4096"]
    assert list(P.q_primes) == g["q_primes"] and list(P.t_primes) == g["t_primes"]
    assert [R.root_of_unity(8192, q) for q in P.q_primes] == g["psi"]
    assert [P.delta % q for q in P.q_primes] == g["delta_mod_q"]
    assert P.relin_digits == g["relin_digits"] == 14
    assert P.fresh_noise == g["fresh_noise"]
    assert R.ntt_primes(4096, 30, 15) == g["aux_primes_15"]
    P8 = H.p8192_params()
    assert list(P8.q_primes) == golden["p8192"]["q_primes"]
    assert list(P8.t_primes) == golden["p8192"]["t_primes"]
    Ps = H.default_params(512, plain_bits=17)
    assert list(Ps.q_primes) == golden["p512"]["q_primes"]


def test_known_answer_wrap():
    # reference tests/test_ring.py:49-53: x^3 * x = -1 in Z_17[x]/(x^4+1)
    a = np.array([0, 0, 0, 1], dtype=np.uint64)
    b = np.array([0, 1, 0, 0], dtype=np.uint64)
    assert R.negacyclic_mul_mod(a, b, 17).tolist() == [16, 0, 0, 0]


def test_ntt_forward_matches_reference(golden):
    for case in golden["ntt"]:
        n, p = case["n"], case["p"]
        a = R.sample_uniform(p, n, np.random.default_rng(case["seed"]))
        assert digest(a) == case["in"]
        plan = R.NttPlan(n, p)
        fa = plan.forward(a)
        assert digest(fa) == case["fwd"], (n, p)
        assert [int(v) for v in fa[:4]] == case["fwd_head"]
        assert np.array_equal(np.asarray(plan.inverse(fa), dtype=np.uint64), np.asarray(a, dtype=np.uint64))


def test_ntt_eval_layout():
    # out[k] = a(psi^(2 bitrev(k) + 1))
    n, p = 16, R.ntt_primes(16, 18, 1)[0]
    psi = R.root_of_unity(2 * n, p)
    a = R.sample_uniform(p, n, np.random.default_rng(3))
    fa = R.NttPlan(n, p).forward(a)
    for k in range(n):
        x = pow(psi, 2 * R.bitrev(k, 4) + 1, p)
        assert int(fa[k]) == sum(int(c) * pow(x, i, p) for i, c in enumerate(a)) % p


def test_cfg1_keys_and_cpmul_match_reference(golden):
    P = H.default_params(4096)
    g = golden["cfg1"]
    keys = H.keygen(P, g["keygen_seed"])
    assert digest(np.asarray(keys["s"], dtype=np.int64).astype(np.uint64)) == g["sk"]
    assert digest(keys["pk"][0]) == g["pk0"] and digest(keys["pk"][1]) == g["pk1"]
    assert digest(keys["relin"][0][0]) == g["relin0_b"]
    assert digest(keys["relin"][-1][1]) == g["relin13_a"]
    rng = np.random.default_rng(g["rng_seed"])
    c0 = H.ints_to_rns(P, R.sample_uniform(P.q, P.n, rng))
    c1 = H.ints_to_rns(P, R.sample_uniform(P.q, P.n, rng))
    pt = R.sample_uniform(P.t, P.n, rng)
    ct = np.stack([c0, c1])
    assert digest(ct) == g["c_in"] and digest(pt) == g["pt"]
    assert digest(H.cp_mul(P, ct, pt)) == g["cpmul"]
    assert P.cp_mul_noise(P.fresh_noise) == g["cpmul_noise"]
    m = R.sample_uniform(P.t, P.n, rng)
    cte = H.encrypt(P, m, keys["pk"], rng)
    assert digest(m) == g["m"] and digest(cte) == g["enc"]
    prod = H.cp_mul(P, cte, pt)
    assert digest(prod) == g["enc_cpmul"]
    dec = H.decrypt(P, prod, keys["s"])
    assert digest(dec) == g["dec"]
    assert np.array_equal(dec, H.pp_mul(P, m, pt))


def test_ppmul_matches_reference(golden):
    P = H.default_params(4096)
    a = R.sample_uniform(P.t, P.n, np.random.default_rng(55))
    b = R.sample_uniform(P.t, P.n, np.random.default_rng(56))
    assert digest(H.pp_mul(P, a, b)) == golden["ppmul"]["out"]


def test_ccmul_relin_512_matches_reference(golden):
    P = H.default_params(512, plain_bits=17)
    g = golden["ccmul512"]
    keys = H.keygen(P, g["keygen_seed"])
    rng = np.random.default_rng(g["rng_seed"])
    ma = R.sample_uniform(P.t, P.n, rng)
    mb = R.sample_uniform(P.t, P.n, rng)
    ca = H.encrypt(P, ma, keys["pk"], rng)
    cb = H.encrypt(P, mb, keys["pk"], rng)
    assert digest(ca) == g["ca"] and digest(cb) == g["cb"]
    raw = H.cc_mul_raw(P, ca, cb)
    assert digest(raw) == g["raw"]
    rel = H.relinearize(P, raw, keys["relin"])
    assert digest(rel) == g["relin"]
    assert digest(H.decrypt(P, rel, keys["s"])) == g["dec"]


def test_known_answer_products_512():
    """Reference tests/test_he.py:78-87 (Enc(3)*Enc(5) decrypts to 15) and the CPMul
    negacyclic wrap: Enc(x^(n-1)) * x = -1, i.e. t-1 in coefficient 0."""
    P = H.default_params(512, plain_bits=17)
    keys = H.keygen(P, 7)
    rng = np.random.default_rng(8)

    def mono(v, deg):
        m = np.zeros(P.n, dtype=np.uint64)
        m[deg] = v
        return m

    three = H.encrypt(P, mono(3, 0), keys["pk"], rng)
    five = H.encrypt(P, mono(5, 0), keys["pk"], rng)
    out = H.decrypt(P, H.cc_mul(P, three, five, keys["relin"]), keys["s"])
    assert int(out[0]) == 15 and not out[1:].any()
    top = H.encrypt(P, mono(1, P.n - 1), keys["pk"], rng)
    out = H.decrypt(P, H.cp_mul(P, top, mono(1, 1)), keys["s"])
    assert int(out[0]) == P.t - 1 and not out[1:].any()
    # CCAdd of the two fresh ciphertexts decrypts to the plain sum
    out = H.decrypt(P, H._add(P, three, five), keys["s"])
    assert int(out[0]) == 8 and not out[1:].any()


@pytest.mark.slow
def test_ccmul_4096_matches_reference(golden):
    P = H.default_params(4096)
    g = golden["ccmul4096"]
    keys = H.keygen(P, 1)
    rng = np.random.default_rng(g["rng_seed"])
    ma = R.sample_uniform(P.t, P.n, rng)
    mb = R.sample_uniform(P.t, P.n, rng)
    ca = H.encrypt(P, ma, keys["pk"], rng)
    cb = H.encrypt(P, mb, keys["pk"], rng)
    assert digest(ca) == g["ca"]
    raw = H.cc_mul_raw(P, ca, cb)
    assert digest(raw) == g["raw"]
    rel = H.relinearize(P, raw, keys["relin"])
    assert digest(rel) == g["relin"]


def test_serialization_matches_reference(golden):
    import hashlib
    P = H.default_params(4096)
    rng = np.random.default_rng(1234)
    c0 = R.sample_uniform(P.q, P.n, rng)
    blob = R.ring_to_bytes(c0, P.n, P.q)
    assert len(blob) == golden["serial"]["len"]
    assert hashlib.sha256(blob).hexdigest() == golden["serial"]["c0_bytes"]
    back = R.ring_from_bytes(blob, P.n, P.q)
    assert all(int(a) == int(b) for a, b in zip(back, c0))


# ---------------------------------------------------------------- the protocol restatement (oracle/linprot_ref.py)

def _proto_check(case, p, job_id, job):
    import hashlib
    from oracle import linprot_ref as LP
    from oracle import packing_ref as PR
    res = LP.run_protocol(p, job_id, job)
    assert len(res["c2s"]) == case["c2s_len"] and len(res["s2c"]) == case["s2c_len"]
    assert hashlib.sha256(res["c2s"]).hexdigest() == case["c2s"]
    assert hashlib.sha256(res["s2c"]).hexdigest() == case["s2c"]
    signed = PR.centered(job["extract"](res["out"]), p.t)
    assert list(signed.shape) == case["tensor_shape"]
    assert digest(signed.astype(np.uint64)) == case["tensor"]
    return signed


def test_protocol_restatement_matches_reference_transcripts(golden):
    """oracle.linprot_ref + oracle.packing_ref reproduce the reference's two-party precompute-protocol
    transcripts (both directions, every ciphertext byte) for conv, grad-w and FC jobs."""
    from oracle import packing_ref as PR
    from oracle.plainconv import conv2d_multi
    Ps = H.default_params(512, plain_bits=17)
    g = golden["protocol"]["small_conv"]
    x, w = np.array(g["x"]), np.array(g["w"])
    out = _proto_check(g, Ps, "c", PR.conv_job(x, w, 8, 8, 3, 1, 512, Ps.t))
    assert np.array_equal(out, conv2d_multi(x, w, 1))
    g = golden["protocol"]["small_gradw"]
    _proto_check(g, Ps, "g", PR.conv_grad_w_job(np.array(g["x"]), np.array(g["gy"]), 6, 6, 4, 1, 512, Ps.t))
    g = golden["protocol"]["small_fc"]
    x, w = np.array(g["x"]), np.array(g["w"])
    out = _proto_check(g, Ps, "fc", PR.fc_job(x, w, 512, Ps.t))
    assert np.array_equal(out, w @ x)


def test_packing_restatement_plans(golden):
    from oracle import packing_ref as PR
    g = golden["packing"]
    assert list(PR.choose_tiles(64, 64, 5, 4096)) == g["choose_tiles_64_64_5_4_4096"]
    assert PR.plan(28, 28, 5, 0, 4096)["O"] == g["cfg3_plan"]
    assert PR.plan(32, 32, 3, 1, 4096)["O"] == g["cfg4_plan"]
    pl = PR.plan(32, 32, 32, 1, 4096)
    assert [pl["O"], len(pl["tiles"])] == g["cfg4_gw_plan"]
    # reference tests/test_packing.py toy degrees: 2x2 input -> {0,1,3,4}, 2x2 kernel -> {4,3,1,0}
    pl = PR.plan(2, 2, 2, 0, 16)
    assert sorted(np.nonzero(PR.pack_input(np.array([[1, 2], [3, 4]]), pl, 97)[0])[0].tolist()) == [0, 1, 3, 4]
    k = PR.pack_kernel(np.array([[1, 2], [3, 4]]), pl, 97)
    assert [int(k[d]) for d in (4, 3, 1, 0)] == [1, 2, 3, 4]
