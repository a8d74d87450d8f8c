"""GPU parity of the ring mirror (ring.py surface) against the oracle."""
import numpy as np
import pytest

from conftest import has_gpu
from oracle import ring_ref as R

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def test_wrap_and_monomials():
    from paper_2409_16675_b200 import ring
    from paper_2409_16675_b200.ring import RingElem, RingParams
    P = RingParams(4, 17)
    x3 = RingElem.monomial(P, 1, 3)
    x1 = RingElem.monomial(P, 1, 1)
    assert ring.ring_mul(x3, x1).to_ints() == [16, 0, 0, 0]
    for n in (8, 16, 32):
        p = R.ntt_primes(n, 18, 1)[0]
        Pn = RingParams(n, p)
        for i in range(n):
            a = RingElem.monomial(Pn, 3, i)
            b = RingElem.monomial(Pn, 5, (i * 7) % n)
            want = R.negacyclic_mul_mod(np.asarray(a.coeffs), np.asarray(b.coeffs), p)
            assert ring.ring_mul(a, b).coeffs.tolist() == [int(v) for v in want]


def test_cipher_ring_ops_match_oracle():
    from paper_2409_16675_b200 import ring
    from paper_2409_16675_b200.params import default_he_params
    from paper_2409_16675_b200.ring import RingElem
    P = default_he_params(4096)
    q = P.q
    rng = np.random.default_rng(5)
    a = RingElem.random(P.cipher_ring, rng)
    b = RingElem.random(P.cipher_ring, rng)
    ai = [int(v) for v in a.coeffs]
    bi = [int(v) for v in b.coeffs]
    assert [int(v) for v in ring.ring_add(a, b).coeffs[:64]] == [(x + y) % q for x, y in zip(ai[:64], bi[:64])]
    assert [int(v) for v in ring.ring_sub(a, b).coeffs[:64]] == [(x - y) % q for x, y in zip(ai[:64], bi[:64])]
    assert [int(v) for v in ring.ring_neg(a).coeffs[:64]] == [(-x) % q for x in ai[:64]]
    c = 123456789123456789123
    assert [int(v) for v in ring.ring_scalar_mul(a, c).coeffs[:64]] == [x * c % q for x in ai[:64]]
    prod = ring.ring_mul(a, b)
    want = R.ring_mul_rns(R.to_rns(ai, P.cipher_ring.primes), R.to_rns(bi, P.cipher_ring.primes), P.cipher_ring.primes)
    assert np.array_equal(prod.data.cpu().numpy().astype(np.uint64), want)
    # from_ints with signed big ints
    vals = [(-1) ** i * (i * 10 ** 40 + 7) for i in range(P.n)]
    e = RingElem.from_ints(P.cipher_ring, np.array(vals, dtype=object))
    assert [int(v) for v in e.coeffs[:32]] == [v % q for v in vals[:32]]


def test_plain_ring_ops_and_ntt_surface():
    from paper_2409_16675_b200 import ring
    from paper_2409_16675_b200.ring import RingElem, RingParams
    from paper_2409_16675_b200.params import default_plain_params
    T = default_plain_params(4096)
    rng = np.random.default_rng(8)
    a = RingElem.random(T, rng)
    b = RingElem.random(T, rng)
    t = T.modulus
    av, bv = a.coeffs.astype(object), b.coeffs.astype(object)
    assert np.array_equal(ring.ring_add(a, b).coeffs, ((av + bv) % t).astype(np.uint64))
    assert np.array_equal(ring.ring_sub(a, b).coeffs, ((av - bv) % t).astype(np.uint64))
    assert np.array_equal(ring.ring_scalar_mul(a, 10 ** 15 + 3).coeffs, (av * (10 ** 15 + 3) % t).astype(np.uint64))
    # single-prime eval-domain surface (ring.py:549-584)
    p = R.ntt_primes(32, 18, 1)[0]
    P = RingParams(32, p)
    x = RingElem.random(P, rng)
    y = RingElem.random(P, rng)
    fx = ring.ntt_forward(x)
    assert fx.domain == "eval"
    assert np.array_equal(fx.coeffs, R.NttPlan(32, p).forward(x.coeffs))
    assert ring.ntt_inverse(fx) == x
    ptw = ring.ntt_inverse(ring.pointwise_mul(fx, ring.ntt_forward(y)))
    assert ptw == ring.ring_mul(x, y)
    with pytest.raises(ring.NttUnavailableError):
        ring.ntt_forward(RingElem.zeros(RingParams(8, 19)))
    with pytest.raises(ring.ParamsMismatchError):
        ring.ring_add(RingElem.zeros(RingParams(4, 17)), RingElem.zeros(RingParams(4, 97)))


def test_eval_addend_is_scaled_forward_ntt():
    """ctb_eval_addend(x) == NTT(x) * N^-1 mod p (canonical), the K3 mask-product form."""
    import torch
    from paper_2409_16675_b200 import _lib
    from paper_2409_16675_b200.device import RnsContext, _ptr, _stream
    from paper_2409_16675_b200.params import default_he_params
    P = default_he_params(4096)
    ctx = RnsContext.get(P.n, P.cipher_ring.primes, P.plain_ring.primes)
    p = torch.tensor(P.cipher_ring.primes, dtype=torch.int64, device="cuda").view(1, -1, 1)
    x = (torch.randint(0, 1 << 62, (3, ctx.L, P.n), device="cuda") % p).to(torch.int32)
    ev = torch.empty_like(x)
    _lib.check(ctx._lib.ctb_eval_addend(ctx._h, 0, _ptr(x), _ptr(ev), 3, _stream()), "ctb_eval_addend")
    f = torch.empty_like(x)
    _lib.check(ctx._lib.ctb_ntt_forward(ctx._h, 0, _ptr(x), _ptr(f), 3, _stream()), "ctb_ntt_forward")
    ninv = torch.tensor([pow(P.n, -1, q) for q in P.cipher_ring.primes], dtype=torch.int64, device="cuda").view(1, -1, 1)
    expect = (f.to(torch.int64) * ninv) % p
    assert torch.equal(ev.to(torch.int64), expect)


def test_linear_addend_is_eval_addend_in_thread_major_layout():
    """ctb_linear_addend = ctb_eval_addend permuted into ctb_linear_online's internal layout: 16-byte
    chunk c of transform thread t at chunk c * (N/16) + t, where thread t holds the 16-word eval
    block f(t) (at N = 4096 f rotates the low 5 thread bits: ntt.cuh pass_thread)."""
    import torch
    from paper_2409_16675_b200 import _lib
    from paper_2409_16675_b200.device import RnsContext, _ptr, _stream
    from paper_2409_16675_b200.params import default_he_params
    P = default_he_params(4096)
    ctx = RnsContext.get(P.n, P.cipher_ring.primes, P.plain_ring.primes)
    p = torch.tensor(P.cipher_ring.primes, dtype=torch.int64, device="cuda").view(1, -1, 1)
    x = (torch.randint(0, 1 << 62, (3, ctx.L, P.n), device="cuda") % p).to(torch.int32)
    ev, lin = torch.empty_like(x), torch.empty_like(x)
    _lib.check(ctx._lib.ctb_eval_addend(ctx._h, 0, _ptr(x), _ptr(ev), 3, _stream()), "ctb_eval_addend")
    _lib.check(ctx._lib.ctb_linear_addend(ctx._h, 0, _ptr(x), _ptr(lin), 3, _stream()), "ctb_linear_addend")
    threads = P.n // 16
    t = torch.arange(threads)
    f = (t & ~31) | ((t << 1) & 30) | ((t >> 4) & 1)
    c = torch.arange(4)
    src = (4 * f[None, :] + c[:, None]).reshape(-1)           # eval chunk of strip chunk c*threads + t
    want = ev.view(3, ctx.L, P.n // 4, 4)[:, :, src.cuda()].reshape(3, ctx.L, P.n)
    assert torch.equal(lin, want)


def test_cpmul_host_pipeline_matches_device_path_threads():
    """RnsContext.cpmul_host (pinned host buffers, chunked H2D / CPMul / D2H on 3 streams, the
    bench's e2e leg) equals ctb_cpmul on device buffers, also from two threads at once."""
    import threading
    import torch
    from paper_2409_16675_b200.device import RnsContext
    from paper_2409_16675_b200.params import default_he_params
    P = default_he_params(4096)
    ctx = RnsContext.get(P.n, P.cipher_ring.primes, P.plain_ring.primes)
    p = torch.tensor(P.cipher_ring.primes, dtype=torch.int64).view(1, 1, -1, 1)
    g = torch.Generator().manual_seed(5)
    results, errors = {}, []

    def run(tag, B, chunks):
        try:
            ct = (torch.randint(0, 1 << 62, (B, 2, ctx.L, P.n), generator=g) % p).to(torch.int32)
            pt = torch.randint(0, P.t, (B, P.n), dtype=torch.int64, generator=g)
            want = ctx.cpmul(ct.cuda(), pt.cuda()).cpu()
            out = torch.empty_like(ct).pin_memory()
            ctx.cpmul_host(ct.pin_memory(), pt.pin_memory(), out, chunks=chunks)
            torch.cuda.current_stream().synchronize()
            results[tag] = torch.equal(out, want)
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)

    run("single", 37, 5)
    ts = [threading.Thread(target=run, args=(f"t{i}", 24 + i, 3 + i)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    assert results == {"single": True, "t0": True, "t1": True}


@pytest.mark.parametrize("bits,count", [(31, 2), (20, 3), (31, 1)])
def test_small_moduli_outside_the_plain_context(bits, count):
    """Moduli < 2^63 whose factorisation is not a 1-2 prime (< 2^30) plain context: two primes below
    2^31 (ntt_primes(n, 31, 2), allowed by the reference's cap), three 20-bit primes, one 31-bit prime.
    Elementwise ops and products go through the residues and back (ring.py _small_op)."""
    from paper_2409_16675_b200 import ring
    from paper_2409_16675_b200.ring import RingElem, RingParams
    n = 256
    primes = R.ntt_primes(n, bits, count)
    m = 1
    for p in primes:
        m *= p
    P = RingParams(n, m, tuple(primes))
    rng = np.random.default_rng(bits * 10 + count)
    a = RingElem.random(P, rng)
    b = RingElem.random(P, rng)
    ai = [int(v) for v in a.coeffs]
    bi = [int(v) for v in b.coeffs]
    assert ring.ring_add(a, b).to_ints() == [(x + y) % m for x, y in zip(ai, bi)]
    assert ring.ring_sub(a, b).to_ints() == [(x - y) % m for x, y in zip(ai, bi)]
    assert ring.ring_neg(a).to_ints() == [(-x) % m for x in ai]
    c = 987654321987
    assert ring.ring_scalar_mul(a, c).to_ints() == [x * c % m for x in ai]
    want = R.crt_combine(R.ring_mul_rns(R.to_rns(ai, primes), R.to_rns(bi, primes), primes), primes)
    assert ring.ring_mul(a, b).to_ints() == [int(v) for v in want]


def _pack_ref(vals, bits):
    """Host reference of the dense packed format: value j at bits [j*bits, (j+1)*bits), LE words."""
    acc, nb, out = 0, 0, []
    for v in vals:
        acc |= int(v) << nb
        nb += bits
        while nb >= 32:
            out.append(acc & 0xFFFFFFFF)
            acc >>= 32
            nb -= 32
    if nb:
        out.append(acc & 0xFFFFFFFF)
    return np.array(out, dtype=np.uint64).astype(np.uint32)


@pytest.mark.parametrize("bits,word", [(30, 4), (17, 4), (32, 4), (50, 8), (35, 8), (64, 8), (1, 4)])
def test_bits_pack_roundtrip_matches_host_reference(bits, word):
    import torch
    from paper_2409_16675_b200.device import RnsContext
    from paper_2409_16675_b200.params import default_he_params
    P = default_he_params(4096)
    ctx = RnsContext.get(P.n, P.cipher_ring.primes, P.plain_ring.primes)
    rng = np.random.default_rng(bits)
    count = 4096 * 3 + 32
    hi = 1 << bits
    vals = rng.integers(0, hi, size=count, dtype=np.uint64) if bits < 64 else rng.integers(0, 1 << 63, size=count, dtype=np.uint64) * 2 + 1
    vals[:3] = [0, hi - 1, hi >> 1] if bits < 64 else [0, (1 << 64) - 1, 1 << 63]
    dt = torch.int32 if word == 4 else torch.int64
    x = torch.from_numpy(vals.astype(np.uint32 if word == 4 else np.uint64).view(np.int32 if word == 4 else np.int64)).cuda()
    packed = ctx.pack_bits(x, bits)
    assert np.array_equal(packed.cpu().numpy().view(np.uint32), _pack_ref(vals.tolist(), bits))
    back = ctx.unpack_bits(packed, bits, (count,), dt)
    assert torch.equal(back, x)


def test_cpmul_host_packed_equals_device_path():
    import torch
    from paper_2409_16675_b200.device import RnsContext
    from paper_2409_16675_b200.params import default_he_params
    P = default_he_params(4096)
    qs = P.cipher_ring.primes
    ctx = RnsContext.get(P.n, qs, P.plain_ring.primes)
    B = 37
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    ct = torch.empty((B, 2, len(qs), P.n), dtype=torch.int32, device="cuda")
    for i, q in enumerate(qs):
        ct[:, :, i] = torch.randint(0, q, (B, 2, P.n), generator=g, device="cuda").to(torch.int32)
    pt = torch.randint(0, P.t, (B, P.n), generator=g, device="cuda")
    want = ctx.cpmul(ct, pt)
    ctp = ctx.pack_bits(ct, ctx.q_bits).cpu().pin_memory()
    ptp = ctx.pack_bits(pt, ctx.t_bits).cpu().pin_memory()
    outp = torch.empty_like(ctp).pin_memory()
    assert ctx.q_bits == 30 and ctx.t_bits == 50
    assert ctp.numel() * 4 == B * 2 * len(qs) * P.n * 30 // 8
    ctx.cpmul_host_packed(ctp, ptp, outp, B, chunks=4)
    torch.cuda.synchronize()
    assert torch.equal(ctx.unpack_bits(outp.cuda(), 30, tuple(want.shape), torch.int32), want)
