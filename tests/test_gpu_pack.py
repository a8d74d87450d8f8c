"""The encode / decode kernels (csrc/pack.cu: ctb_pack_gather, ctb_plain_scatter; rns.cu:
ctb_decrypt_round_extract) against the oracle's restatement of the reference packing
(oracle/packing_ref.py <- packing.py:407-605), bit for bit, including multi-tile plans, negative
and out-of-range values, the fused masking, the stride lowering and empty batches."""
import numpy as np
import pytest
import torch

from conftest import has_gpu
from oracle import packing_ref as PR

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

SHAPES = [  # (H, W, kernel, pad, n)
    (28, 28, 5, 0, 4096),    # cfg3 (1 tile)
    (32, 32, 3, 1, 4096),    # cfg4 fwd / gx
    (32, 32, 32, 1, 4096),   # cfg4 grad-w (the gradient as the kernel)
    (64, 64, 5, 4, 4096),    # multi-tile (choose_tiles known answer (56, 64))
    (40, 40, 3, 1, 512),     # many tiles
    (8, 8, 3, 1, 8192),
]


@pytest.fixture(scope="module")
def plain4096():
    from paper_2409_16675_b200.params import default_plain_params
    return default_plain_params(4096)


def _plain(n):
    from paper_2409_16675_b200.params import default_plain_params
    return default_plain_params(n)


@pytest.mark.parametrize("H,W,h,pad,n", SHAPES)
def test_conv_pack_and_extract_match_oracle(H, W, h, pad, n):
    from paper_2409_16675_b200 import packing
    from paper_2409_16675_b200.ring import context_of
    pr = _plain(n)
    t = pr.modulus
    rng = np.random.default_rng(H * 100 + h)
    shape = packing.ConvShape(H, W, h, pad)
    plan = packing.plan_correlated(shape, n)
    pl = PR.plan(H, W, h, pad, n)
    assert plan.row_stride == pl["O"] and [(tt.row0, tt.col0) for tt in plan.tiles] == pl["tiles"]
    x = rng.integers(-(1 << 40), 1 << 40, size=(3, H, W))
    x[0, 0, 0] = -(1 << 62)
    x[0, 0, 1] = t + 5                      # above the modulus: reduced like RingElem.from_ints
    got = packing.pack_input_batch(torch.as_tensor(x, device="cuda"), plan, pr).cpu().numpy()
    for c in range(3):
        assert np.array_equal(got[c].astype(np.uint64), PR.pack_input(x[c], pl, t))
    w = rng.integers(-300, 300, size=(2, h, h))
    gw = packing.pack_kernel_batch(torch.as_tensor(w, device="cuda"), plan, pr).cpu().numpy()
    for k in range(2):
        assert np.array_equal(gw[k].astype(np.uint64), PR.pack_kernel(w[k], pl, t))
    # decode: random product polynomials, residues and centred
    T = plan.num_tiles
    prods = rng.integers(0, t, size=(2, T, n), dtype=np.uint64)
    dev = torch.as_tensor(prods.astype(np.int64), device="cuda")
    res = packing.extract_batch(dev, plan, pr).cpu().numpy()
    cen = packing.extract_batch(dev, plan, pr, centered=True).cpu().numpy()
    for k in range(2):
        want = PR.extract(prods[k], pl)
        assert np.array_equal(res[k].astype(np.uint64), want)
        assert np.array_equal(cen[k], PR.centered(want, t))
    # the same decode with the fused mask subtraction of ctb_plain_scatter
    sub = rng.integers(0, t, size=(2 * T, n), dtype=np.uint64)
    out = packing.conv_output_side(plan, n, 2, (2,))
    got = packing.scatter(context_of(pr), dev.reshape(-1, n), out,
                          sub=torch.as_tensor(sub.astype(np.int64), device="cuda"), centered=True).cpu().numpy()
    diff = ((prods.reshape(-1, n).astype(object) - sub.astype(object)) % t).astype(np.uint64).reshape(2, T, n)
    for k in range(2):
        assert np.array_equal(got[k], PR.centered(PR.extract(diff[k], pl), t))


def test_masked_gather_and_job_builders_match_oracle(plain4096):
    from paper_2409_16675_b200 import linprot, packing
    from paper_2409_16675_b200.ring import context_of
    t, n = plain4096.modulus, 4096
    rng = np.random.default_rng(9)
    x = rng.integers(0, 256, size=(3, 32, 32))
    w = rng.integers(-128, 128, size=(4, 3, 3, 3))
    job = linprot.conv_job("j", x, w, packing.ConvShape(32, 32, 3, 1), plain4096)
    ref = PR.conv_job(x, w, 32, 32, 3, 1, n, t)
    assert [job.shape.n_x, job.shape.n_w, job.shape.n_out] == [ref["n_x"], ref["n_w"], ref["n_out"]]
    assert [tuple(s) for s in job.shape.sites] == ref["sites"]
    r_x = torch.as_tensor(rng.integers(0, t, size=(ref["n_x"], n), dtype=np.uint64).astype(np.int64), device="cuda")
    r_w = torch.as_tensor(rng.integers(0, t, size=(ref["n_w"], n), dtype=np.uint64).astype(np.int64), device="cuda")
    mx, mw = job.masked(context_of(plain4096), r_x, r_w)     # one gather per side: packed + masked
    assert np.array_equal(job.x_plain.cpu().numpy().astype(np.uint64), ref["x"])
    assert np.array_equal(job.w_plain.cpu().numpy().astype(np.uint64), ref["w"])
    for m, plain, r in ((mx, ref["x"], r_x), (mw, ref["w"], r_w)):
        want = (plain.astype(object) - r.cpu().numpy().astype(object)) % t
        assert np.array_equal(m.cpu().numpy().astype(np.uint64), want.astype(np.uint64))
    # grad-w and fc / outer builders
    xg = rng.integers(0, 256, size=(2, 6, 6))
    gy = rng.integers(-128, 128, size=(3, 4, 4))
    job = linprot.conv_grad_w_job("g", xg, gy, packing.ConvShape(6, 6, 4, 1), plain4096)
    ref = PR.conv_grad_w_job(xg, gy, 6, 6, 4, 1, n, t)
    assert [tuple(s) for s in job.shape.sites] == ref["sites"]
    assert np.array_equal(job.x_plain.cpu().numpy().astype(np.uint64), ref["x"])
    assert np.array_equal(job.w_plain.cpu().numpy().astype(np.uint64), ref["w"])
    for out_dim, in_dim in ((5, 40), (1000, 10), (3, 4096)):
        xf = rng.integers(-200, 200, size=in_dim)
        wf = rng.integers(-200, 200, size=(out_dim, in_dim))
        job = linprot.fc_job("fc", xf, wf, plain4096)
        ref = PR.fc_job(xf, wf, n, t)
        assert np.array_equal(job.x_plain.cpu().numpy().astype(np.uint64), ref["x"])
        assert np.array_equal(job.w_plain.cpu().numpy().astype(np.uint64), ref["w"])
        prods = rng.integers(0, t, size=(ref["n_out"], n), dtype=np.uint64)
        got = job.extract(torch.as_tensor(prods.astype(np.int64), device="cuda")).cpu().numpy()
        assert np.array_equal(got.astype(np.uint64), ref["extract"](prods))
    # outer product g x^T: g[r] at degree r*in (packing.py:589-599), output rows r*in .. r*in+in-1
    g = rng.integers(-50, 50, size=700)
    xo = rng.integers(-50, 50, size=9)
    job = linprot.outer_job("o", g, xo, plain4096)
    cap = n // 9
    wp = job.w_plain.cpu().numpy()
    for r in range(700):
        grp, k = divmod(r, cap)
        assert wp[grp, k * 9] == g[r] % t
    prods = rng.integers(0, t, size=(job.shape.n_out, n), dtype=np.uint64)
    got = job.extract(torch.as_tensor(prods.astype(np.int64), device="cuda")).cpu().numpy()
    want = np.stack([prods[r // cap, (r % cap) * 9:(r % cap) * 9 + 9] for r in range(700)])
    assert np.array_equal(got.astype(np.uint64), want)


def test_batched_fc_and_outer_jobs_stay_inside_each_image(plain4096):
    """Batched FC / outer jobs (one job for B images) equal the per-image jobs block by block; the
    last row group of an image (fewer than cap rows, packing.py:581-583) neither reads nor writes
    the next image."""
    from paper_2409_16675_b200 import linprot
    t, n = plain4096.modulus, 4096
    rng = np.random.default_rng(12)
    xs = rng.integers(-50, 50, size=(3, 10))
    wf = rng.integers(-50, 50, size=(1000, 10))            # cap 409: groups of 409, 409, 182 rows
    gs = rng.integers(-50, 50, size=(3, 700))
    xo = rng.integers(-50, 50, size=(3, 9))                # cap 455: groups of 455, 245
    for big, singles in ((linprot.fc_job_batch("fb", xs, wf, plain4096),
                          [linprot.fc_job("f", xs[b], wf, plain4096) for b in range(3)]),
                         (linprot.outer_job_batch("ob", gs, xo, plain4096),
                          [linprot.outer_job("o", gs[b], xo[b], plain4096) for b in range(3)])):
        G = singles[0].shape.n_w
        assert big.shape.n_w == 3 * G and big.shape.n_out == 3 * G
        prods = rng.integers(0, t, size=(3 * G, n), dtype=np.uint64)
        got = big.extract(torch.as_tensor(prods.astype(np.int64), device="cuda")).cpu().numpy()
        for b, one in enumerate(singles):
            assert torch.equal(big.w_plain[b * G:(b + 1) * G], one.w_plain)
            assert torch.equal(big.x_plain[b], one.x_plain[0])
            want = one.extract(torch.as_tensor(prods[b * G:(b + 1) * G].astype(np.int64), device="cuda"))
            assert np.array_equal(got[b], want.cpu().numpy())


def test_decrypt_extract_epilogue_equals_unfused(plain4096):
    """ctb_decrypt_round_extract == ctb_decrypt_round, then c - p, then the extraction, then the
    centring; also with the stride-2 extraction map (= the full output subsampled)."""
    from paper_2409_16675_b200 import he, packing
    P = he.default_he_params(4096)
    ev = he.He(P)
    keys = ev.keygen(5)
    rng = np.random.default_rng(6)
    plan = packing.plan_correlated(packing.ConvShape(32, 32, 3, 1), 4096)
    m = torch.as_tensor(rng.integers(0, P.t, size=(6, 4096), dtype=np.uint64).astype(np.int64), device="cuda")
    cts = ev.encrypt_many(m, keys, np.random.default_rng(7))
    p = torch.as_tensor(rng.integers(0, P.t, size=(6, 4096), dtype=np.uint64).astype(np.int64), device="cuda")
    dec = ev.decrypt_values(cts, keys)
    assert torch.equal(dec, m)
    for stride in (1, 2):
        out = packing.conv_output_side(plan, 4096, 6, (6,), stride)
        fused = ev.decrypt_extract(cts, keys, out, sub=p, centered=True)
        diff = torch.remainder(dec - p, P.t)
        full = packing.extract_batch(diff.view(6, 1, 4096), plan, P.plain_ring, centered=True)
        assert torch.equal(fused, full[:, ::stride, ::stride])
        resid = ev.decrypt_extract(cts, keys, out, sub=p, centered=False)
        assert torch.equal(resid, torch.remainder(full, P.t)[:, ::stride, ::stride])


def test_empty_and_malformed(plain4096):
    from paper_2409_16675_b200 import _lib, packing
    from paper_2409_16675_b200.ring import context_of
    ctx = context_of(plain4096)
    plan = packing.plan_correlated(packing.ConvShape(8, 8, 3, 1), 4096)
    side = packing.conv_input_side(torch.zeros((0, 8, 8), dtype=torch.int64, device="cuda"), plan, 4096)
    assert side.n_polys == 0
    assert packing.gather(ctx, side).shape == (0, 4096)
    with pytest.raises(packing.PackingError):
        packing.gather(ctx, packing.conv_input_side(torch.zeros((1, 8, 8), dtype=torch.int64, device="cuda"),
                                                    plan, 4096), r=torch.zeros((2, 4096), dtype=torch.int64,
                                                                               device="cuda"))
    lib = _lib.load()
    assert lib.ctb_pack_gather(ctx._h, None, 0, None, 0, None, None, None, None, None, 1, None) == -1
    assert lib.ctb_plain_scatter(ctx._h, None, None, None, 0, None, None, 0, 0, None, 1, None) == -1
    assert lib.ctb_pack_gather(ctx._h, None, 0, None, 0, None, None, None, None, None, 0, None) == 0


@pytest.mark.parametrize("params_name", ["p4096", "p8192"])
def test_encrypt_gather_equals_pack_then_encrypt(params_name):
    """ctb_encrypt_gather (the packing read inside the encryption kernel) == ctb_pack_gather followed
    by ctb_encrypt, ciphertext for ciphertext, at 32- and 64-bit limbs (same numpy draws)."""
    from paper_2409_16675_b200 import he, linprot, packing
    P = he.default_he_params(4096) if params_name == "p4096" else he.p8192_he_params()
    ev = he.He(P)
    keys = ev.keygen(2)
    rng = np.random.default_rng(31)
    x = rng.integers(-300, 300, size=(3, 9, 9))
    w = rng.integers(-128, 128, size=(4, 3, 3, 3))
    job = linprot.conv_job("e", x, w, packing.ConvShape(9, 9, 3, 1), P.plain_ring)
    for side, plain in ((job.x_side, job.x_plain), (job.w_side, job.w_plain)):
        a = ev.encrypt_many(side, keys, np.random.default_rng(8))
        b = ev.encrypt_many(plain, keys, np.random.default_rng(8))
        assert torch.equal(a.data, b.data)
        gen_a, gen_b = torch.Generator(device="cuda"), torch.Generator(device="cuda")
        gen_a.manual_seed(3)
        gen_b.manual_seed(3)
        assert torch.equal(ev.encrypt_many(side, keys, gen_a).data, ev.encrypt_many(plain, keys, gen_b).data)
    fc = linprot.fc_job("f", rng.integers(-9, 9, size=50), rng.integers(-9, 9, size=(700, 50)), P.plain_ring)
    a = ev.encrypt_many(fc.w_side, keys, np.random.default_rng(4))
    assert torch.equal(a.data, ev.encrypt_many(fc.w_plain, keys, np.random.default_rng(4)).data)


def test_descriptor_bounds_are_enforced_per_element():
    """Map rows beyond n_maps, sources beyond src_len and destinations beyond dst_len contribute
    zero / are dropped instead of reading or writing out of bounds (ctb_pack_gather,
    ctb_plain_scatter, ctb_decrypt_round_extract share the rule)."""
    from paper_2409_16675_b200 import he, packing
    P = he.default_he_params(4096)
    ev = he.He(P)
    ctx = ev.ctx
    n = P.n
    maps = torch.full((2, n), -1, dtype=torch.int32, device="cuda")
    maps[0, :8] = torch.arange(8, dtype=torch.int32)
    maps[1, :8] = torch.arange(8, dtype=torch.int32) + 4
    src = torch.arange(1, 11, dtype=torch.int64, device="cuda") * -3      # 10 values, negative
    kind = torch.tensor([0, 1, 5], dtype=torch.int32, device="cuda")      # kind 5: no such row
    base = torch.tensor([0, 0, 0], dtype=torch.int64, device="cuda")
    side = packing.Gather(src, maps, kind, base)
    out = packing.gather(ctx, side).cpu().numpy()
    t = P.t
    assert [int(v) for v in out[0, :8]] == [(-3 * (i + 1)) % t for i in range(8)]
    # row 1 reads src[4..11]: the last two are past src_len -> 0
    assert [int(v) for v in out[1, :8]] == [(-3 * (i + 5)) % t for i in range(6)] + [0, 0]
    assert not out[2].any() and not out[:, 8:].any()
    # scatter: destinations past dst_len are dropped (rows 0 and 1 write disjoint ranges)
    maps2 = maps.clone()
    maps2[1, :8] = torch.arange(8, dtype=torch.int32) + 8
    vals = torch.arange(3 * n, dtype=torch.int64, device="cuda").view(3, n) % t
    res = packing.scatter(ctx, vals, packing.Scatter(maps2, kind, base, (10,))).cpu().numpy()
    assert res.tolist() == list(range(8)) + [n, n + 1]
