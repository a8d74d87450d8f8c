"""Reference protocol/pool/hygiene tests (pkg/tests/test_linprot.py, test_he.py)
restated for the device path (rlwe backend: the device path has no clear backend)."""
import numpy as np
import pytest

from conftest import has_gpu
from oracle.plainconv import conv2d

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def p512():
    from paper_2409_16675_b200 import he
    plain = he.default_plain_params(512, 17, 2)
    return he.HeParams(he.default_cipher_params(512, plain.modulus), plain)


def evaluators(params):
    from paper_2409_16675_b200 import he
    cli, srv = he.He(params), he.He(params)
    return cli, srv, cli.keygen(3)


def run_b(params, job):
    from paper_2409_16675_b200 import channel, linprot
    cli, srv, keys = evaluators(params)

    def c(end):
        linprot.setup_client(end, cli, keys)
        return linprot.linear_b_client(end, cli, keys, np.random.default_rng(1), job)

    def s(end):
        pks = linprot.setup_server(end, srv)
        linprot.linear_b_server(end, srv, pks)

    ce, se = channel.inproc_pair()
    res, _ = channel.run_pair(c, s, ce, se)
    return res, cli, srv


def run_pre(params, job, count=1, capture=False):
    from paper_2409_16675_b200 import channel, linprot
    cli, srv, keys = evaluators(params)
    cpool, spool = linprot.TriplePool(), linprot.TriplePool()

    def c(end):
        linprot.setup_client(end, cli, keys)
        linprot.precompute_offline_client(end, cli, keys, np.random.default_rng(2), job.shape, count, cpool)
        return linprot.precompute_online_client(end, cli, keys, np.random.default_rng(4), job, cpool)

    def s(end):
        pks = linprot.setup_server(end, srv)
        linprot.precompute_offline_server(end, srv, pks, spool)
        linprot.precompute_online_server(end, srv, pks, spool)

    ce, se = channel.inproc_pair(capture=capture)
    res, _ = channel.run_pair(c, s, ce, se)
    return res, cli, srv, keys, ce, cpool, spool


def signed(t, modulus):
    from paper_2409_16675_b200 import packing
    return packing.to_signed_tensor(t, modulus).cpu().numpy().astype(np.int64)


def test_protocol_b_equals_precompute_equals_plain(p512, rng):
    from paper_2409_16675_b200 import linprot, packing
    shape = packing.ConvShape(8, 8, 3, 1)
    x = rng.integers(-40, 40, size=(1, 8, 8))
    w = rng.integers(-9, 9, size=(1, 1, 3, 3))
    rb, _, srv_b = run_b(p512, linprot.conv_job("c", x, w, shape, p512.plain_ring))
    rp, *_ = run_pre(p512, linprot.conv_job("c", x, w, shape, p512.plain_ring))
    plain = conv2d(x[0], w[0, 0], 1)
    assert np.array_equal(signed(rb.tensor[0], p512.t), plain)
    assert np.array_equal(signed(rp.tensor[0], p512.t), plain)
    assert srv_b.meter.count("CCMul", "online") == 1


def test_identity_kernel_and_toy(p512, rng):
    from paper_2409_16675_b200 import linprot, packing
    x = rng.integers(-50, 50, size=(1, 4, 4))
    res, *_ = run_pre(p512, linprot.conv_job("ident", x, np.ones((1, 1, 1, 1), dtype=np.int64),
                                              packing.ConvShape(4, 4, 1, 0), p512.plain_ring))
    assert np.array_equal(signed(res.tensor[0], p512.t), x[0])
    x = rng.integers(-20, 20, size=(1, 2, 2))
    w = rng.integers(-9, 9, size=(1, 1, 2, 2))
    res, *_ = run_pre(p512, linprot.conv_job("toy", x, w, packing.ConvShape(2, 2, 2, 1), p512.plain_ring))
    assert np.array_equal(signed(res.tensor[0], p512.t), conv2d(x[0], w[0, 0], 1))


def test_fc_outer_affine_and_bn(p512, rng):
    from paper_2409_16675_b200 import channel, linprot
    W = rng.integers(-30, 30, size=(4, 4))
    x = rng.integers(-30, 30, size=4)
    res, *_ = run_pre(p512, linprot.fc_job("fc", x, W, p512.plain_ring))
    assert np.array_equal(signed(res.tensor, p512.t), W @ x)
    g = rng.integers(-9, 9, size=3)
    res, *_ = run_pre(p512, linprot.outer_job("outer", g, x, p512.plain_ring))
    assert np.array_equal(signed(res.tensor, p512.t), np.outer(g, x))
    xa = rng.integers(-100, 100, size=(5, 5))
    res, *_ = run_pre(p512, linprot.affine_job("bn", xa, 7, p512.plain_ring))
    assert np.array_equal(signed(res.tensor, p512.t), xa * 7)
    beta = rng.integers(-10, 10, size=(5, 5))
    cli, srv, keys = evaluators(p512)

    def c(end):
        linprot.setup_client(end, cli, keys)
        return linprot.bn_affine_client(end, cli, keys, np.random.default_rng(1), "bn", xa, 3, beta)

    def s(end):
        linprot.linear_b_server(end, srv, linprot.setup_server(end, srv))

    ce, se = channel.inproc_pair()
    r, _ = channel.run_pair(c, s, ce, se)
    assert np.array_equal(r.tensor, xa * 3 + beta)


def test_online_meters_per_site(p512, rng):
    from paper_2409_16675_b200 import linprot, packing
    x = rng.integers(-5, 5, size=(1, 3, 3))
    w = rng.integers(-5, 5, size=(1, 1, 2, 2))
    job = linprot.conv_job("m", x, w, packing.ConvShape(3, 3, 2, 0), p512.plain_ring)
    nsites = len(job.shape.sites)
    _, cli, srv, *_ = run_pre(p512, job)
    assert srv.meter.count("CCMul", "online") == 0
    assert srv.meter.count("CCMul", "offline") == nsites
    assert srv.meter.count("Relin", "offline") == nsites
    assert srv.meter.count("CPMul", "online") == 2 * nsites
    assert srv.meter.count("PPMul", "online") == nsites
    assert srv.meter.count("CCAdd", "online") >= 2 * nsites


def test_pool_discipline_and_mask_product(p512, rng, tmp_path):
    from paper_2409_16675_b200 import channel, linprot, ring
    from paper_2409_16675_b200.ring import RingElem
    cli, srv, keys = evaluators(p512)
    cpool, spool = linprot.TriplePool(), linprot.TriplePool()
    js = linprot.JobShape("L", 1, 1, 1, ((0, 0, 0),))

    def c(end):
        linprot.setup_client(end, cli, keys)
        linprot.precompute_offline_client(end, cli, keys, np.random.default_rng(0), js, 2, cpool)

    def s(end):
        pks = linprot.setup_server(end, srv)
        linprot.precompute_offline_server(end, srv, pks, spool)

    ce, se = channel.inproc_pair()
    channel.run_pair(c, s, ce, se)
    # persistence round trip
    linprot.save_server_pool(spool, srv, str(tmp_path / "s.pool"))
    linprot.save_client_pool(cpool, str(tmp_path / "c.pool"))   # reference signature (linprot.py:550)
    spool2 = linprot.load_server_pool(srv, str(tmp_path / "s.pool"))
    cpool2 = linprot.load_client_pool(p512.plain_ring, str(tmp_path / "c.pool"))   # linprot.py:565
    assert spool2.available("L") == 2 and cpool2.available("L") == 2
    b1, b2 = cpool.take("L"), cpool2.take("L")
    assert np.array_equal(b1.r_x.cpu().numpy(), b2.r_x.cpu().numpy())
    p1, p2 = spool.take("L"), spool2.take("L")
    # the server's slot decrypts to r_x * r_w (test secret key)
    expect = ring.ring_mul(RingElem(p512.plain_ring, b1.r_x[0]), RingElem(p512.plain_ring, b1.r_w[0]))
    assert srv.decrypt(p1.slots[0], keys) == expect
    assert srv.decrypt(p2.slots[0], keys) == expect
    with pytest.raises(linprot.SingleUseViolationError):
        b1.consume()
    cpool.take("L")
    with pytest.raises(linprot.PoolExhaustedError):
        cpool.take("L")


def test_transcript_hygiene(p512, rng):
    from paper_2409_16675_b200 import linprot, packing, ring
    from paper_2409_16675_b200.ring import RingElem
    x = rng.integers(100, 1 << 15, size=(1, 4, 4))
    w = rng.integers(100, 1 << 15, size=(1, 1, 2, 2))
    job = linprot.conv_job("h", x, w, packing.ConvShape(4, 4, 2, 1), p512.plain_ring)
    _, cli, srv, keys, ce, *_ = run_pre(p512, job, capture=True)
    blob = bytes(ce.stats.transcript["client"]) + bytes(ce.stats.transcript["server"])
    assert ring.ring_to_bytes(job.x_polys[0])[5:] not in blob
    assert ring.ring_to_bytes(job.w_polys[0])[5:] not in blob
    assert cli.secret_key_to_bytes(keys)[5:] not in blob
    r_x = RingElem.random(p512.plain_ring, np.random.default_rng(2))
    masked = ring.ring_sub(job.x_polys[0], r_x)
    assert ring.ring_to_bytes(masked)[5:] in blob


def test_meter_relin_exactly_once_n64():
    # reference tests/test_he.py:117-130 at N = 64
    from paper_2409_16675_b200 import he
    from paper_2409_16675_b200.ring import RingElem
    plain = he.default_plain_params(64, prime_bits=17, primes=2)
    params = he.HeParams(he.default_cipher_params(64, plain.modulus), plain)
    ev = he.He(params)
    keys = ev.keygen(3)
    rng = np.random.default_rng(0)
    a = ev.encrypt(RingElem.random(plain, rng), keys, rng)
    b = ev.encrypt(RingElem.random(plain, rng), keys, rng)
    ev.cc_mul(a, b, keys)
    assert ev.meter.count("CCMul") == 1 and ev.meter.count("Relin") == 1
    ev.cp_mul(a, RingElem.zeros(plain))
    assert ev.meter.count("CPMul") == 1 and ev.meter.count("Relin") == 1


def test_depth_budget_validation():
    from paper_2409_16675_b200 import he
    from paper_2409_16675_b200.params import RingParams, ntt_primes
    plain = he.default_plain_params(64, prime_bits=17, primes=2)
    thin = ntt_primes(64, 30, 2)
    with pytest.raises(ValueError):
        he.HeParams(RingParams(64, thin[0] * thin[1], primes=tuple(thin)), plain).check_depth_budget()


def test_c_abi_errors_and_empty_batches():
    import ctypes
    import torch
    from paper_2409_16675_b200 import _lib
    from paper_2409_16675_b200.device import RnsContext
    from paper_2409_16675_b200.params import default_he_params
    lib = _lib.load()
    P = default_he_params(4096)
    ctx = RnsContext.get(P.n, P.cipher_ring.primes, P.plain_ring.primes)
    assert lib.ctb_cpmul(ctx._h, None, None, None, 1, None) == _lib.CTB_ERR_ARG
    assert b"ctb_cpmul" in lib.ctb_last_error()
    assert lib.ctb_ntt_forward(ctx._h, 7, None, None, 1, None) == _lib.CTB_ERR_ARG
    h = ctypes.c_void_p()
    rc = lib.ctb_ctx_create(ctypes.byref(h), 4096, _lib.u64_array([1073692673 + 2]), 1, _lib.u64_array([]), 0, 16)
    assert rc == _lib.CTB_ERR_ARG and b"1 mod 2N" in lib.ctb_last_error()
    empty = torch.empty((0, 2, ctx.L, P.n), dtype=torch.int32, device="cuda")
    assert ctx.cpmul(empty, torch.empty((0, P.n), dtype=torch.int64, device="cuda")).shape[0] == 0
    with pytest.raises(ValueError):
        ctx.cpmul(empty[:, :1], torch.empty((0, P.n), dtype=torch.int64, device="cuda"))


def _ccmul_sum_case(p512, rng, job):
    """Offline mask products of one job via the fused path; returned as host residues."""
    from paper_2409_16675_b200 import linprot
    from paper_2409_16675_b200.he import CiphertextBatch
    cli, srv, keys = evaluators(p512)
    pks = srv.public_keys_from_bytes(cli.public_keys_to_bytes(keys))
    js = job.shape
    r = linprot._plain_random(cli, js.n_x + js.n_w, np.random.default_rng(7))
    cts = cli.encrypt_many(r, keys, np.random.default_rng(8))
    fresh = srv.params.fresh_noise
    rx = CiphertextBatch(cts.data[:js.n_x], fresh, cts.backend_tag, cts._cipher)
    rw = CiphertextBatch(cts.data[js.n_x:], fresh, cts.backend_tag, cts._cipher)
    out = linprot._sites_ccmul_sum(srv, pks, rx, rw, js)
    # per-site reference through the single-CCMul API, CCAdd per slot
    per = srv.cc_mul_many(
        CiphertextBatch(rx.data[[s[0] for s in js.sites]].contiguous(), fresh, rx.backend_tag, rx._cipher),
        CiphertextBatch(rw.data[[s[1] for s in js.sites]].contiguous(), fresh, rw.backend_tag, rw._cipher), pks)
    ref = [None] * js.n_out
    for k, (_, _, o) in enumerate(js.sites):
        c = per[k]
        ref[o] = c if ref[o] is None else srv.cc_add(ref[o], c)
    return out, ref


def test_ccmul_sum_matches_per_site_and_chunks(p512, rng):
    """ctb_ccmul_sum == per-site cc_mul + relinearize + CCAdd (he.py:434-439, linprot.py:407-427),
    single-chunk and with the multi-chunk path forced (CTB_SITE_CHUNK=2 in a subprocess)."""
    import os
    import subprocess
    import sys
    import torch
    from paper_2409_16675_b200 import linprot, packing
    x = rng.integers(0, 50, size=(2, 6, 6))
    w = rng.integers(-9, 9, size=(3, 2, 3, 3))
    job = linprot.conv_job("cs", x, w, packing.ConvShape(6, 6, 3, 1), p512.plain_ring)
    out, ref = _ccmul_sum_case(p512, rng, job)
    assert all(torch.equal(out.data[o], c.data) for o, c in enumerate(ref))
    code = (
        "import numpy as np, torch, sys; sys.path.insert(0, 'tests'); "
        "import test_gpu_protocol_extra as t; from paper_2409_16675_b200 import he, linprot, packing; "
        "plain = he.default_plain_params(512, 17, 2); "
        "P = he.HeParams(he.default_cipher_params(512, plain.modulus), plain); "
        "rng = np.random.default_rng(3); x = rng.integers(0, 50, size=(2, 6, 6)); "
        "w = rng.integers(-9, 9, size=(3, 2, 3, 3)); "
        "job = linprot.conv_job('cs', x, w, packing.ConvShape(6, 6, 3, 1), P.plain_ring); "
        "out, ref = t._ccmul_sum_case(P, rng, job); "
        "print('OK' if all(torch.equal(out.data[o], c.data) for o, c in enumerate(ref)) else 'BAD')")
    env = dict(os.environ, CTB_SITE_CHUNK="2")
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
    assert res.stdout.strip().endswith("OK"), res.stdout + res.stderr


def test_c_abi_fused_entry_errors():
    """ctb_ccmul_sum / ctb_linear_online reject out-of-range sites and short workspaces."""
    import ctypes
    import torch
    from paper_2409_16675_b200 import _lib
    from paper_2409_16675_b200.device import RnsContext, _ptr, _stream
    from paper_2409_16675_b200.params import default_he_params
    P = default_he_params(4096)
    ctx = RnsContext.get(P.n, P.cipher_ring.primes, P.plain_ring.primes)
    lib = _lib.load()
    ct = torch.zeros((2, 2, ctx.L, P.n), dtype=torch.int32, device="cuda")
    sites = (ctypes.c_uint32 * 3)(0, 5, 0)   # w index 5 out of range
    keys = torch.zeros((14, 2, ctx.L, P.n), dtype=torch.int32, device="cuda")
    out = torch.empty((1, 2, ctx.L, P.n), dtype=torch.int32, device="cuda")
    wsb = int(lib.ctb_ccmul_sum_workspace_bytes(ctx._h, 2, 2, 1, 1, 1))
    work = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    rc = lib.ctb_ccmul_sum(ctx._h, _ptr(ct), 2, _ptr(ct), 2, sites, 1, 1, _ptr(keys), _ptr(out), _ptr(work), wsb,
                           _stream())
    assert rc == _lib.CTB_ERR_ARG and b"out of range" in lib.ctb_last_error()
    good = (ctypes.c_uint32 * 3)(0, 1, 0)
    rc = lib.ctb_ccmul_sum(ctx._h, _ptr(ct), 2, _ptr(ct), 2, good, 1, 1, _ptr(keys), _ptr(out), _ptr(work), 16,
                           _stream())
    assert rc == _lib.CTB_ERR_ARG and b"workspace" in lib.ctb_last_error()
    mx = torch.zeros((2, P.n), dtype=torch.int64, device="cuda")
    wsl = int(lib.ctb_linear_online_workspace_bytes(ctx._h, 2, 2, 1, 1))
    work2 = torch.empty(wsl, dtype=torch.uint8, device="cuda")
    outp = torch.empty((1, P.n), dtype=torch.int64, device="cuda")
    rc = lib.ctb_linear_online(ctx._h, _ptr(ct), 2, _ptr(ct), 2, _ptr(mx), _ptr(mx), sites, 1, 1, None, 0,
                               _ptr(out), _ptr(outp), _ptr(work2), _stream())
    assert rc == _lib.CTB_ERR_ARG and b"out of range" in lib.ctb_last_error()


def test_server_rejects_inconsistent_jobs(p512):
    """The server validates the declared JobShape against what arrived: too few blobs,
    out-of-range sites or a pool entry with the wrong slot count raise LinProtError before any
    device buffer is sized from the header."""
    import torch
    from paper_2409_16675_b200 import linprot
    cli, srv, keys = evaluators(p512)
    pks = srv.public_keys_from_bytes(cli.public_keys_to_bytes(keys))
    pool = linprot.TriplePool()
    js = linprot.JobShape("L", 2, 1, 1, ((0, 0, 0), (1, 0, 0)))
    with pytest.raises(linprot.LinProtError):
        linprot.precompute_online_server(None, srv, pks, pool, blobs=[b"pre", js.to_bytes(), b"", b""])
    with pytest.raises(linprot.LinProtError):
        linprot.linear_b_server(None, srv, pks, blobs=[b"b", js.to_bytes(), b""])
    bad = linprot.JobShape("L", 1, 1, 1, ((0, 0, 3),))
    with pytest.raises(linprot.LinProtError):
        linprot.linear_b_server(None, srv, pks, blobs=[b"b", bad.to_bytes(), b"", b""])
    # a pool entry whose slot count differs from the job's
    cts = cli.encrypt_many(torch.zeros((2, p512.n), dtype=torch.int64, device="cuda"), keys, np.random.default_rng(1))
    pool.add(linprot.MaskProduct("L", cts))
    blobs = [b"pre", js.to_bytes()] + cli.batch_to_bytes(cts) + cli.batch_to_bytes(cts)[:1] \
        + cli.plain_to_bytes(torch.zeros((3, p512.n), dtype=torch.int64, device="cuda"))
    with pytest.raises(linprot.LinProtError):
        linprot.precompute_online_server(None, srv, pks, pool, blobs=blobs)
