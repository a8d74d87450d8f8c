"""GPU parity: NTT / ring_mul / CPMul / PPMul through the C ABI versus the oracle
(pinned to the reference by tests/golden).  Bit-exact integer equality."""
import numpy as np
import pytest

from _util import digest
from conftest import has_gpu
from oracle import he_ref as H
from oracle import ring_ref as R

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def _t(arr, dtype):
    import torch
    return torch.from_numpy(np.ascontiguousarray(np.asarray(arr, dtype=np.int64))).to(dtype).cuda()


def _np(t):
    return t.cpu().numpy().astype(np.uint64)


@pytest.fixture(scope="module")
def p4096():
    return H.default_params(4096)


@pytest.fixture(scope="module")
def ctx4096(p4096):
    from paper_2409_16675_b200.device import RnsContext
    return RnsContext.get(p4096.n, p4096.q_primes, p4096.t_primes)


def test_ntt_forward_per_limb_matches_reference(golden):
    import torch
    from paper_2409_16675_b200.device import RnsContext
    for case in golden["ntt"]:
        n, p = case["n"], case["p"]
        a = R.sample_uniform(p, n, np.random.default_rng(case["seed"]))
        ctx = RnsContext.get(n, [p])
        x = _t(a, ctx.dtype()).reshape(1, 1, n)
        fa = ctx.ntt_forward(x)
        torch.cuda.synchronize()
        assert digest(_np(fa).reshape(-1)) == case["fwd"], (n, p)
        back = ctx.ntt_inverse(fa)
        assert np.array_equal(_np(back).reshape(-1), np.asarray(a, dtype=np.uint64))


@pytest.mark.parametrize("logn", [2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13])
@pytest.mark.parametrize("bits", [30, 50])
def test_ntt_all_degrees_match_oracle(logn, bits):
    from paper_2409_16675_b200.device import RnsContext
    n = 1 << logn
    if bits == 30 and logn < 4:
        primes = R.ntt_primes(n, 20, 2)
    else:
        primes = R.ntt_primes(n, bits, 2)
    ctx = RnsContext.get(n, primes)
    rng = np.random.default_rng(logn * 100 + bits)
    a = np.stack([np.stack([R.sample_uniform(p, n, rng) for p in primes]) for _ in range(3)])
    fa = _np(ctx.ntt_forward(_t(a, ctx.dtype())))
    for b in range(3):
        for i, p in enumerate(primes):
            want = np.asarray(R.NttPlan(n, p).forward(a[b, i]), dtype=np.uint64)
            assert np.array_equal(fa[b, i], want), (logn, bits, b, i)
    back = _np(ctx.ntt_inverse(_t(fa.astype(np.int64), ctx.dtype())))
    assert np.array_equal(back, a.astype(np.uint64))


@pytest.mark.parametrize("logn,bits", [(6, 30), (9, 30), (12, 30), (13, 30), (12, 50), (13, 50), (12, 36), (10, 44)])
def test_ring_mul_matches_oracle(logn, bits):
    from paper_2409_16675_b200.device import RnsContext
    n = 1 << logn
    primes = R.ntt_primes(n, bits, 3)
    ctx = RnsContext.get(n, primes)
    rng = np.random.default_rng(7 + logn)
    a = np.stack([np.stack([R.sample_uniform(p, n, rng) for p in primes]) for _ in range(2)])
    b = np.stack([np.stack([R.sample_uniform(p, n, rng) for p in primes]) for _ in range(2)])
    got = _np(ctx.ring_mul(_t(a, ctx.dtype()), _t(b, ctx.dtype())))
    assert np.array_equal(got, R.ring_mul_rns(a, b, primes))
    # broadcast one operand
    got1 = _np(ctx.ring_mul(_t(a, ctx.dtype()), _t(b[:1], ctx.dtype())))
    assert np.array_equal(got1, R.ring_mul_rns(a, np.broadcast_to(b[:1], a.shape), primes))


def test_cpmul_cfg1_matches_reference(golden, p4096, ctx4096):
    g = golden["cfg1"]
    P = p4096
    rng = np.random.default_rng(g["rng_seed"])
    c0 = H.ints_to_rns(P, R.sample_uniform(P.q, P.n, rng))
    c1 = H.ints_to_rns(P, R.sample_uniform(P.q, P.n, rng))
    pt = R.sample_uniform(P.t, P.n, rng)
    ct = np.stack([c0, c1])[None]
    out = _np(ctx4096.cpmul(_t(ct, ctx4096.dtype()), _t(pt[None], __import__("torch").int64)))
    assert digest(out[0]) == g["cpmul"]


def test_cpmul_batch_matches_oracle(p4096, ctx4096):
    import torch
    P = p4096
    B = 24
    rng = np.random.default_rng(99)
    ct = np.stack([np.stack([H.ints_to_rns(P, R.sample_uniform(P.q, P.n, rng)) for _ in range(2)]) for _ in range(B)])
    pt = np.stack([R.sample_uniform(P.t, P.n, rng) for _ in range(B)])
    # include the lift boundary: exactly t//2 and t//2 + 1, 0 and t-1
    pt[0, :4] = [P.t // 2, P.t // 2 + 1, 0, P.t - 1]
    got = _np(ctx4096.cpmul(_t(ct, ctx4096.dtype()), _t(pt, torch.int64)))
    for b in range(B):
        assert np.array_equal(got[b], H.cp_mul(P, ct[b], pt[b])), b
    # in-place
    x = _t(ct, ctx4096.dtype())
    ctx4096.cpmul(x, _t(pt, torch.int64), out=x)
    assert np.array_equal(_np(x), got)


def test_cpmul_p8192_matches_restatement():
    import torch
    from paper_2409_16675_b200.device import RnsContext
    P = H.p8192_params()
    ctx = RnsContext.get(P.n, P.q_primes, P.t_primes)
    assert ctx.word_bytes() == 8
    rng = np.random.default_rng(8192)
    B = 2
    ct = np.stack([np.stack([np.stack([R.sample_uniform(q, P.n, rng) for q in P.q_primes]) for _ in range(2)])
                   for _ in range(B)])
    pt = np.stack([R.sample_uniform(P.t, P.n, rng) for _ in range(B)])
    got = _np(ctx.cpmul(_t(ct.astype(np.int64), torch.int64), _t(pt, torch.int64)))
    for b in range(B):
        assert np.array_equal(got[b], H.cp_mul(P, ct[b], pt[b]))


def test_ppmul_matches_reference(golden, p4096, ctx4096):
    import torch
    P = p4096
    a = R.sample_uniform(P.t, P.n, np.random.default_rng(55))
    b = R.sample_uniform(P.t, P.n, np.random.default_rng(56))
    got = _np(ctx4096.pp_mul(_t(a[None], torch.int64), _t(b[None], torch.int64)))
    assert digest(got[0]) == golden["ppmul"]["out"]


def test_encrypted_cpmul_decrypts(golden, p4096, ctx4096):
    """Encrypt on the oracle, CPMul on the GPU, decrypt on the oracle: the
    decrypted product equals the plain ring product and the reference digest."""
    import torch
    g = golden["cfg1"]
    P = p4096
    keys = H.keygen(P, g["keygen_seed"])
    rng = np.random.default_rng(g["rng_seed"])
    for _ in range(3):
        R.sample_uniform(P.q, P.n, rng) if _ < 2 else None
    pt = R.sample_uniform(P.t, P.n, rng)
    m = R.sample_uniform(P.t, P.n, rng)
    cte = H.encrypt(P, m, keys["pk"], rng)
    out = _np(ctx4096.cpmul(_t(cte[None], ctx4096.dtype()), _t(pt[None], torch.int64)))[0]
    assert digest(out) == g["enc_cpmul"]
    assert digest(H.decrypt(P, out, keys["s"])) == g["dec"]


@pytest.mark.parametrize("logn", [6, 12, 13])
def test_fp64_butterflies_extreme_inputs(logn):
    """50-bit limbs run FP64 butterflies (ntt.cuh): all-(p-1), alternating 0/(p-1) and
    single-spike inputs on the largest primes below 2^50 must match the exact oracle."""
    from paper_2409_16675_b200.device import RnsContext
    n = 1 << logn
    primes = R.ntt_primes(n, 50, 3)
    ctx = RnsContext.get(n, primes)
    pv = np.asarray(primes, dtype=np.uint64)[:, None]
    full = np.broadcast_to(pv - 1, (3, n))
    alt = np.where(np.arange(n) % 2 == 0, 0, pv - 1).astype(np.uint64)
    spike = np.zeros((3, n), dtype=np.uint64)
    spike[:, n - 1] = (pv - 1)[:, 0]
    a = np.stack([full, alt, spike]).astype(np.uint64)
    fa = _np(ctx.ntt_forward(_t(a, ctx.dtype())))
    for b in range(3):
        for i, p in enumerate(primes):
            assert np.array_equal(fa[b, i], np.asarray(R.NttPlan(n, p).forward(a[b, i]), dtype=np.uint64)), (b, i)
    back = _np(ctx.ntt_inverse(_t(fa.astype(np.int64), ctx.dtype())))
    assert np.array_equal(back, a)
    got = _np(ctx.ring_mul(_t(a, ctx.dtype()), _t(a[::-1].copy(), ctx.dtype())))
    assert np.array_equal(got, R.ring_mul_rns(a, a[::-1].copy(), primes))


@pytest.mark.parametrize("which", ["p4096", "p8192"])
def test_cpmul_empty_and_maximum_inputs(which):
    """Edge cases: an empty batch is a no-op (reference cp_mul is per-object, so the batched
    boundary's B=0 must not launch or fault), and every residue at q_i - 1 with every plaintext
    coefficient at t - 1 (largest operands of each modular product) matches the oracle."""
    import torch
    from paper_2409_16675_b200.device import RnsContext
    P = H.default_params(4096) if which == "p4096" else H.p8192_params()
    ctx = RnsContext.get(P.n, P.q_primes, P.t_primes)
    L = len(P.q_primes)
    empty = torch.empty((0, 2, L, P.n), dtype=ctx.dtype(), device="cuda")
    out = ctx.cpmul(empty, torch.empty((0, P.n), dtype=torch.int64, device="cuda"))
    assert out.shape == (0, 2, L, P.n)
    ct = np.stack([np.stack([np.full(P.n, q - 1, dtype=np.uint64) for q in P.q_primes])] * 2)[None]
    pts = [np.full(P.n, P.t - 1, dtype=np.uint64), np.full(P.n, P.t // 2 + 1, dtype=np.uint64)]
    for pt in pts:
        got = _np(ctx.cpmul(_t(ct, ctx.dtype()), _t(pt[None], torch.int64)))
        assert np.array_equal(got[0], H.cp_mul(P, ct[0], pt))
        fa = ctx.ntt_forward(_t(ct[:, 0], ctx.dtype()))
        back = _np(ctx.ntt_inverse(fa))
        assert np.array_equal(back, ct[:, 0])
