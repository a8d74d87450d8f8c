"""Ciphertext-level parity where round 1 only checked decrypted outputs.

* cfg4 (one image of the BASELINE conv layer, N=4096 default parameters): the device client + server
  reproduce, byte for byte in both directions, the REAL reference's two-party precompute-protocol
  transcripts of the layer's forward, weight-gradient and input-gradient jobs
  (tests/golden/make_golden_cfg4.py; lowering train.py:478-494).  The transcripts carry every
  encrypted input, mask ciphertext, masked plaintext and output slot ciphertext, so this pins
  k_encrypt, ctb_ccmul_sum (per-site tensoring + exact rounding + relinearisation + CCAdd),
  ctb_linear_online and the decrypt path on the cfg4 shapes.
* N=8192 / 3 x 50-bit limbs (cfg2b / cfg5 parameters, which the reference cannot construct): the
  same protocol against the oracle restatement's transcripts (tests/golden/make_golden_p8192.py),
  i.e. the u64-limb instantiations of the fused server kernels residue for residue.
"""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from _util import digest
from conftest import has_gpu
from test_gpu_protocol import run_pre

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

GOLD = Path(__file__).resolve().parent / "golden"


def _check(case, params, job):
    from paper_2409_16675_b200 import packing
    res, stats, srv = run_pre(params, job)
    tr = stats.transcript
    assert len(tr["client"]) == case["c2s_len"] and len(tr["server"]) == case["s2c_len"]
    assert hashlib.sha256(bytes(tr["client"])).hexdigest() == case["c2s"], "client->server bytes differ"
    assert hashlib.sha256(bytes(tr["server"])).hexdigest() == case["s2c"], "server->client bytes differ"
    signed = packing.to_signed_tensor(res.tensor, params.t).cpu().numpy().astype(np.int64)
    assert list(signed.shape) == case["tensor_shape"]
    assert digest(signed.astype(np.uint64)) == case["tensor"]
    return signed, srv


@pytest.fixture(scope="module")
def cfg4():
    g = json.loads((GOLD / "golden_cfg4.json").read_text())
    rng = np.random.default_rng(4)
    x = rng.integers(0, 256, size=(3, 32, 32))
    w = rng.integers(-128, 128, size=(64, 3, 3, 3))
    gy = rng.integers(-128, 128, size=(64, 32, 32))
    return g["cases"], x, w, gy


@pytest.mark.parametrize("name", ["fwd", "gw", "gx"])
def test_cfg4_image_transcripts_match_reference(cfg4, name):
    from paper_2409_16675_b200 import he, linprot, packing
    from oracle.plainconv import conv2d_multi
    cases, x, w, gy = cfg4
    P = he.default_he_params(4096)
    pr = P.plain_ring
    if name == "fwd":
        job = linprot.conv_job("cfg4_fwd", x, w, packing.ConvShape(32, 32, 3, 1), pr)
        want = conv2d_multi(x, w, 1)
    elif name == "gw":
        job = linprot.conv_grad_w_job("cfg4_gw", x, gy, packing.ConvShape(32, 32, 32, 1), pr)
        from oracle.plainconv import conv2d
        want = np.stack([np.stack([conv2d(x[ci], gy[co], 1) for ci in range(3)]) for co in range(64)])
    else:
        wrot = np.flip(w, axis=(2, 3)).transpose(1, 0, 2, 3).copy()
        job = linprot.conv_job("cfg4_gx", gy, wrot, packing.ConvShape(32, 32, 3, 1), pr)
        want = conv2d_multi(gy, wrot, 1)
    case = cases[name]
    js = job.shape
    assert [js.n_x, js.n_w, js.n_out, len(js.sites)] == case["js"]
    out, srv = _check(case, P, job)
    assert srv.meter.snapshot()["counts"] == case["server_counts"]
    assert np.array_equal(out, want)


@pytest.fixture(scope="module")
def p8192():
    from paper_2409_16675_b200 import he
    g = json.loads((GOLD / "golden_p8192.json").read_text())
    P = he.p8192_he_params()
    assert list(P.cipher_ring.rns_primes) == g["params"]["q_primes"]
    assert list(P.plain_ring.rns_primes) == g["params"]["t_primes"]
    return P, g["cases"]


def test_p8192_conv_protocol_matches_restatement(p8192):
    from paper_2409_16675_b200 import linprot, packing
    from oracle.plainconv import conv2d_multi
    P, cases = p8192
    c = cases["conv"]
    x, w = np.array(c["x"]), np.array(c["w"])
    out, _ = _check(c, P, linprot.conv_job("conv", x, w, packing.ConvShape(8, 8, 3, 1), P.plain_ring))
    assert np.array_equal(out, conv2d_multi(x, w, 1))


def test_p8192_gradw_protocol_matches_restatement(p8192):
    from paper_2409_16675_b200 import linprot, packing
    P, cases = p8192
    c = cases["gradw"]
    _check(c, P, linprot.conv_grad_w_job("gradw", np.array(c["x"]), np.array(c["gy"]), packing.ConvShape(6, 6, 4, 1),
                                         P.plain_ring))


def test_p8192_fc_protocol_matches_restatement(p8192):
    from paper_2409_16675_b200 import linprot
    P, cases = p8192
    c = cases["fc"]
    x, w = np.array(c["x"]), np.array(c["w"])
    out, _ = _check(c, P, linprot.fc_job("fc", x, w, P.plain_ring))
    assert np.array_equal(out, w @ x)


def _run_b(params, job, keygen_seed=3, online_seed=4):
    from paper_2409_16675_b200 import channel, he, linprot
    cli, srv = he.He(params, he.BACKEND_RLWE), he.He(params, he.BACKEND_RLWE)
    keys = cli.keygen(keygen_seed)

    def client(end):
        linprot.setup_client(end, cli, keys)
        return linprot.linear_b_client(end, cli, keys, np.random.default_rng(online_seed), job)

    def server(end):
        pks = linprot.setup_server(end, srv)
        linprot.linear_b_server(end, srv, pks)

    ce, se = channel.inproc_pair(capture=True)
    res, _ = channel.run_pair(client, server, ce, se)
    return res, ce.stats, srv


@pytest.mark.parametrize("name", ["conv", "fc"])
def test_protocol_b_transcripts_match_reference(name):
    """CryptoTrain-B (direct per-site CCMul on the server, linprot.py:352-379): the device client +
    server reproduce the reference transcripts byte for byte (tests/golden/make_golden_extra.py)."""
    from paper_2409_16675_b200 import he, linprot, packing
    g = json.loads((GOLD / "golden_extra.json").read_text())["protocol_b"][name]
    plain = he.default_plain_params(512, 17, 2)
    Ps = he.HeParams(he.default_cipher_params(512, plain.modulus), plain)
    x, w = np.array(g["x"]), np.array(g["w"])
    if name == "conv":
        job = linprot.conv_job("bc", x, w, packing.ConvShape(8, 8, 3, 1), Ps.plain_ring)
    else:
        job = linprot.fc_job("bf", x, w, Ps.plain_ring)
    res, stats, srv = _run_b(Ps, job)
    tr = stats.transcript
    assert len(tr["client"]) == g["c2s_len"] and len(tr["server"]) == g["s2c_len"]
    assert hashlib.sha256(bytes(tr["client"])).hexdigest() == g["c2s"]
    assert hashlib.sha256(bytes(tr["server"])).hexdigest() == g["s2c"]
    signed = packing.to_signed_tensor(res.tensor, Ps.t).cpu().numpy().astype(np.int64)
    assert digest(signed.astype(np.uint64)) == g["tensor"]
    assert srv.meter.snapshot()["counts"] == g["server_counts"]
