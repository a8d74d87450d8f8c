"""Full BASELINE sizes through size-independent properties (the CPU oracle is
too slow for 4096 ciphertexts at once): cfg2a / cfg2b batched CPMul with
monomial plaintexts equals the exact negacyclic rotation of every residue,
a seeded sample is bit-exact against the oracle, and repeated/in-place
launches agree."""
import numpy as np
import pytest

from conftest import has_gpu
from oracle import he_ref as H
from oracle import ring_ref as R

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def _rotate(ct, k, primes):
    """ct [..., L, N] * x^k (negacyclic) exactly."""
    n = ct.shape[-1]
    out = np.roll(ct, k, axis=-1).astype(np.int64)
    qs = np.array(primes, dtype=np.int64)[:, None]
    if k:
        out[..., :k] = (qs - out[..., :k]) % qs
    return out.astype(np.uint64)


@pytest.mark.parametrize("which", ["p4096", "p8192"])
def test_cpmul_full_batch_properties(which):
    import torch
    from paper_2409_16675_b200.device import RnsContext
    from paper_2409_16675_b200.params import default_he_params, p8192_he_params
    P = default_he_params(4096) if which == "p4096" else p8192_he_params()
    qs = P.cipher_ring.primes
    ctx = RnsContext.get(P.n, qs, P.plain_ring.primes)
    B, n = 4096, P.n
    g = torch.Generator(device="cuda")
    g.manual_seed(77)
    ct = torch.empty((B, 2, len(qs), n), dtype=ctx.dtype(), device="cuda")
    for i, q in enumerate(qs):
        ct[:, :, i, :] = torch.randint(0, q, (B, 2, n), generator=g, device="cuda", dtype=torch.int64).to(ctx.dtype())
    # monomial plaintexts x^k_b (k_b varies per ciphertext): output = rotation of the input
    ks = torch.randint(0, n, (B,), generator=g, device="cuda")
    pt = torch.zeros((B, n), dtype=torch.int64, device="cuda")
    pt[torch.arange(B, device="cuda"), ks] = 1
    out = ctx.cpmul(ct, pt)
    ct_h = ct.cpu().numpy().astype(np.uint64)
    out_h = out.cpu().numpy().astype(np.uint64)
    for b in range(0, B, 97):
        assert np.array_equal(out_h[b], _rotate(ct_h[b], int(ks[b]), qs)), b
    # (-1) * x^k (centred lift of t-1): negated rotation
    pt2 = torch.zeros((B, n), dtype=torch.int64, device="cuda")
    pt2[torch.arange(B, device="cuda"), ks] = P.t - 1
    out2 = ctx.cpmul(ct, pt2).cpu().numpy().astype(np.int64)
    qv = np.array(qs, dtype=np.int64)[:, None]
    for b in range(0, B, 211):
        assert np.array_equal(out2[b], (qv - out_h[b].astype(np.int64)) % qv)
    # random plaintexts: seeded sample bit-exact vs the oracle, repeat and in-place agree
    ptr = torch.randint(0, P.t, (B, n), generator=g, device="cuda", dtype=torch.int64)
    res = ctx.cpmul(ct, ptr)
    again = ctx.cpmul(ct, ptr)
    assert torch.equal(res, again)
    PR = H.default_params(4096) if which == "p4096" else H.p8192_params()
    res_h = res.cpu().numpy().astype(np.uint64)
    pt_h = ptr.cpu().numpy().astype(np.uint64)
    sample = [0, B - 1] + list(np.random.default_rng(5).choice(B, 4 if which == "p4096" else 1, replace=False))
    for b in sample:
        assert np.array_equal(res_h[b], H.cp_mul(PR, ct_h[b], pt_h[b])), b
    x = ct.clone()
    ctx.cpmul(x, ptr, out=x)
    assert torch.equal(x, res)


def test_ntt_full_batch_roundtrip_and_linearity():
    import torch
    from paper_2409_16675_b200.device import RnsContext
    from paper_2409_16675_b200.params import default_he_params
    P = default_he_params(4096)
    qs = P.cipher_ring.primes
    ctx = RnsContext.get(P.n, qs)
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    B = 2048
    a = torch.empty((B, len(qs), P.n), dtype=torch.int32, device="cuda")
    b = torch.empty_like(a)
    for i, q in enumerate(qs):
        a[:, i] = torch.randint(0, q, (B, P.n), generator=g, device="cuda", dtype=torch.int64).int()
        b[:, i] = torch.randint(0, q, (B, P.n), generator=g, device="cuda", dtype=torch.int64).int()
    fa, fb = ctx.ntt_forward(a), ctx.ntt_forward(b)
    assert torch.equal(ctx.ntt_inverse(fa), a)
    qv = torch.tensor(qs, dtype=torch.int64, device="cuda")[:, None]
    s = ((a.long() + b.long()) % qv).int()
    assert torch.equal(ctx.ntt_forward(s), ((fa.long() + fb.long()) % qv).int())   # linearity
