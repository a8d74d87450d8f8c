"""DeviceSecureEngine's non-linear layers are delegated, never computed in the clear by the engine.

relu / maxpool4 must hand their inputs to the injected secure protocol with the reference's
conversions (SecureEngine.relu / maxpool4, train.py:278-290: mpc.from_signed -> session.nonlinear
-> mpc.to_signed).  With the reference importable (this container, not the GPU box) the engine is
driven through the REAL reference OT path: SecureSession.nonlinear against serve_session
(session.py:78-84, 96-125; mpc.client_nonlinear / server_nonlinear).  No GPU is touched: the
non-linear primitives never reach the device path."""
import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")


def _engine(nonlinear, bits=32):
    from paper_2409_16675_b200 import engine
    from paper_2409_16675_b200.params import default_plain_params
    return engine.DeviceSecureEngine(None, plain_ring=default_plain_params(4096), bits=bits, nonlinear=nonlinear)


def test_relu_and_maxpool_delegate_with_reference_conversions():
    from paper_2409_16675_b200 import engine
    calls = []

    def spy(op, values, bits):
        calls.append((op, np.array(values, copy=True), bits))
        return engine.cleartext_nonlinear(op, values, bits)

    eng = _engine(spy)
    x = np.array([[-5, 3], [0, -(1 << 31)]], dtype=np.int64)
    out = eng.relu(x)
    assert np.array_equal(out, np.maximum(x, 0))
    op, vals, bits = calls[-1]
    assert op == "relu" and bits == 32 and vals.dtype == np.uint64
    assert vals.tolist() == [(v + (1 << 32)) % (1 << 32) for v in x.ravel().tolist()]   # mpc.from_signed
    wins = np.array([[1, -7, 4], [9, -2, -4], [-3, -1, 0], [2, -9, 3]], dtype=np.int64)
    assert np.array_equal(eng.maxpool4(wins), wins.max(axis=0))
    assert calls[-1][0] == "maxpool" and calls[-1][1].shape == wins.shape
    assert len(calls) == 2


def test_engine_without_a_protocol_refuses_nonlinear_layers():
    from paper_2409_16675_b200 import engine
    eng = _engine(None)
    with pytest.raises(engine.TrainError):
        eng.relu(np.array([1, -1]))
    with pytest.raises(engine.TrainError):
        eng.maxpool4(np.zeros((4, 2), dtype=np.int64))


def _reference_session_pair():
    sys.path.insert(0, str(REF))
    from privtrain import he, session, transport
    plain = he.default_plain_params(64, prime_bits=17, primes=2)
    params = he.HeParams(he.default_cipher_params(64, plain.modulus), plain)
    return params, he, session, transport


@pytest.mark.skipif(not REF.exists(), reason="the reference (OT protocol) is only present in the build container")
def test_engine_nonlinear_through_reference_secure_session():
    params, he, session, transport = _reference_session_pair()
    rng = np.random.default_rng(5)
    x = rng.integers(-(1 << 20), 1 << 20, size=(3, 4, 4))
    wins = rng.integers(-(1 << 20), 1 << 20, size=(4, 2, 3, 3))
    results = {}

    def client(end):
        sess = session.SecureSession(end, params, he.BACKEND_CLEAR, seed=3)
        sess.setup(keygen_seed=1)
        eng = _engine(sess.nonlinear)
        results["relu"] = eng.relu(x)
        results["pool"] = eng.maxpool4(wins)
        return sess.finish()

    def server(end):
        return session.serve_session(end, params, he.BACKEND_CLEAR)

    ce, se = transport.inproc_pair(timeout=120.0)
    report, _ = transport.run_pair(client, server, ce, se)
    assert np.array_equal(results["relu"], np.maximum(x, 0))
    assert np.array_equal(results["pool"], wins.max(axis=0))
    assert report["comm"]["bytes_by_phase"]["nonlinear"] > 0     # the OT protocol actually ran
