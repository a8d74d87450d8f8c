"""End-to-end protocol parity: the device client + server reproduce the
reference's two-party precompute-protocol transcripts byte for byte (both
directions, pinned by tests/golden from the real reference), the decrypted
tensors and the server's per-op meter counts."""
import hashlib

import numpy as np
import pytest

from _util import digest
from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def run_pre(params, job, keygen_seed=3, offline_seed=2, online_seed=4):
    from paper_2409_16675_b200 import channel, he, linprot
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

    ce, se = channel.inproc_pair(capture=True)
    res, _ = channel.run_pair(client, server, ce, se)
    return res, ce.stats, srv


def check(case, params, job):
    from paper_2409_16675_b200 import packing
    res, stats, srv = run_pre(params, job)
    tr = stats.transcript
    assert len(tr["client"]) == case["c2s_len"] and len(tr["server"]) == case["s2c_len"]
    assert hashlib.sha256(bytes(tr["client"])).hexdigest() == case["c2s"]
    assert hashlib.sha256(bytes(tr["server"])).hexdigest() == case["s2c"]
    signed = packing.to_signed_tensor(res.tensor, params.t).cpu().numpy().astype(np.int64)
    assert list(signed.shape) == case["tensor_shape"]
    assert digest(signed.astype(np.uint64)) == case["tensor"]
    assert srv.meter.snapshot()["counts"] == case["server_counts"]
    return signed


@pytest.fixture(scope="module")
def p512():
    from paper_2409_16675_b200 import he
    plain = he.default_plain_params(512, 17, 2)
    return he.HeParams(he.default_cipher_params(512, plain.modulus), plain)


def test_small_conv_transcript(golden, p512):
    from paper_2409_16675_b200 import linprot, packing
    g = golden["protocol"]["small_conv"]
    x, w = np.array(g["x"]), np.array(g["w"])
    job = linprot.conv_job("c", x, w, packing.ConvShape(8, 8, 3, 1), p512.plain_ring)
    out = check(g, p512, job)
    # and it is the convolution
    from oracle.plainconv import conv2d_multi
    assert np.array_equal(out, conv2d_multi(x, w, 1))


def test_small_gradw_transcript(golden, p512):
    from paper_2409_16675_b200 import linprot, packing
    g = golden["protocol"]["small_gradw"]
    job = linprot.conv_grad_w_job("g", np.array(g["x"]), np.array(g["gy"]), packing.ConvShape(6, 6, 4, 1),
                                  p512.plain_ring)
    check(g, p512, job)


def test_small_fc_transcript(golden, p512):
    from paper_2409_16675_b200 import linprot
    g = golden["protocol"]["small_fc"]
    x, w = np.array(g["x"]), np.array(g["w"])
    out = check(g, p512, linprot.fc_job("fc", x, w, p512.plain_ring))
    assert np.array_equal(out, w @ x)


def test_cfg3_image_transcript(golden):
    from paper_2409_16675_b200 import he, linprot, packing
    P = he.default_he_params(4096)
    g = golden["protocol"]["cfg3_image"]
    rng = np.random.default_rng(3)
    x = rng.integers(0, 256, size=(1, 28, 28))
    w = rng.integers(-128, 128, size=(5, 1, 5, 5))
    out = check(g, P, linprot.conv_job("cfg3", x, w, packing.ConvShape(28, 28, 5, 0), P.plain_ring))
    from oracle.plainconv import conv2d_multi
    assert np.array_equal(out, conv2d_multi(x, w, 0))
