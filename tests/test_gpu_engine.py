"""Trainer-engine parity: the reference trainer's PlainEngine calls (recorded by
tests/golden/make_trainer_golden.py from the real reference) replayed through
engine.DeviceSecureEngine must return identical integers (test_train.py:269-322)."""
from pathlib import Path

import numpy as np
import pytest

from conftest import has_gpu

GOLDEN = Path(__file__).parent / "golden" / "trainer_calls.npz"
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def calls(store, tag):
    for ci in range(int(store[f"{tag}.ncalls"])):
        pre = f"{tag}.call{ci:03d}"
        yield (str(store[f"{pre}.method"]), str(store[f"{pre}.job_id"]), store[f"{pre}.a"], store[f"{pre}.b"],
               store.get(f"{pre}.shape"), store[f"{pre}.out"])


def invoke(eng, method, jid, a, b, shape):
    from paper_2409_16675_b200 import packing
    if method in ("conv_forward", "conv_pairwise"):
        sh = packing.ConvShape(*[int(v) for v in shape])
        return getattr(eng, method)(a, b, sh, job_id=jid)
    if method == "affine":
        return eng.affine(a, int(b), job_id=jid)
    return getattr(eng, method)(a, b, job_id=jid)


def job_for(eng, method, jid, a, b, shape):
    from paper_2409_16675_b200 import linprot, packing
    r = eng.ring
    if method == "conv_forward":
        return linprot.conv_job(jid, a, b, packing.ConvShape(*[int(v) for v in shape]), r)
    if method == "conv_pairwise":
        return linprot.conv_grad_w_job(jid, a, b, packing.ConvShape(*[int(v) for v in shape]), r)
    if method == "fc":
        return linprot.fc_job(jid, b, a, r)
    if method == "outer":
        return linprot.outer_job(jid, a, b, r)
    return linprot.affine_job(jid, a, int(b), r)


@pytest.fixture(scope="module")
def store():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="module")
def params():
    from paper_2409_16675_b200.params import default_he_params
    return default_he_params(4096)


@pytest.mark.parametrize("tag", ["toy", "bn"])
def test_precompute_engine_replays_reference_trainer(store, params, tag):
    from paper_2409_16675_b200 import engine
    sess = engine.DeviceSession(params, engine.PROTOCOL_PRECOMPUTE, seed=5, keygen_seed=2)
    eng = engine.DeviceSecureEngine(sess, params.plain_ring, 32)
    recorded = list(calls(store, tag))
    shapes = {}
    for m, jid, a, b, sh, _ in recorded:
        js = job_for(eng, m, jid, a, b, sh).shape
        shapes.setdefault(jid, (js, 0))
        shapes[jid] = (js, shapes[jid][1] + 1)
    for js, count in shapes.values():
        sess.ensure_offline([js], count)
    for m, jid, a, b, sh, out in recorded:
        got = invoke(eng, m, jid, a, b, sh)
        assert got.dtype == np.int64 and np.array_equal(got, out), (m, jid)
    rep = sess.report()
    assert "online:CCMul" not in rep["server_meter"]["counts"]
    assert rep["server_meter"]["counts"]["offline:CCMul"] > 0
    assert eng.scheme_counts["baseline"] == 0
    assert all(sess.available(jid) == 0 for jid in shapes)


def test_direct_protocol_engine(store, params):
    from paper_2409_16675_b200 import engine
    sess = engine.DeviceSession(params, engine.PROTOCOL_B, seed=7)
    eng = engine.DeviceSecureEngine(sess, params.plain_ring, 32)
    for m, jid, a, b, sh, out in list(calls(store, "toy"))[:6]:
        assert np.array_equal(invoke(eng, m, jid, a, b, sh), out), (m, jid)
    assert sess.report()["server_meter"]["counts"].get("online:CCMul", 0) > 0


def test_engine_errors(params):
    from paper_2409_16675_b200 import engine, linprot, packing
    from paper_2409_16675_b200.params import RingParams, ntt_primes
    sess = engine.DeviceSession(params)
    eng = engine.DeviceSecureEngine(sess)
    with pytest.raises(linprot.PoolExhaustedError):
        eng.conv_forward(np.ones((1, 4, 4), dtype=np.int64), np.ones((1, 1, 3, 3), dtype=np.int64),
                         packing.ConvShape(4, 4, 3, 1), job_id="none")
    small = ntt_primes(4096, 17, 2)
    with pytest.raises(engine.TrainError):
        engine.DeviceSecureEngine(sess, RingParams(4096, small[0] * small[1], primes=tuple(small)), bits=32)
    sess_auto = engine.DeviceSession(params, auto_offline=True)
    eng = engine.DeviceSecureEngine(sess_auto, bits=8)
    with pytest.raises(engine.FixedPointOverflowError):
        eng.affine(np.full((4,), 1000, dtype=np.int64), 1000)


def test_lowerings_and_batch(params, rng):
    from oracle.plainconv import conv2d_multi
    from paper_2409_16675_b200 import engine, linprot, packing
    sess = engine.DeviceSession(params, auto_offline=True)
    eng = engine.DeviceSecureEngine(sess)
    x = rng.integers(-100, 100, size=(2, 10, 10))
    w = rng.integers(-50, 50, size=(3, 2, 3, 3))
    got = eng.conv_forward_strided(x, w, packing.ConvShape(10, 10, 3, 1), 2)
    full = conv2d_multi(x, w, 1)
    assert np.array_equal(got, full[:, ::2, ::2])
    W = rng.integers(-30, 30, size=(5, 9000))
    v = rng.integers(-30, 30, size=9000)
    assert np.array_equal(eng.fc_chunked(W, v), W @ v)
    g = rng.integers(-30, 30, size=3)
    assert np.array_equal(eng.outer_chunked(g, v), np.outer(g, v))
    xs = rng.integers(-100, 100, size=(3, 2, 10, 10))
    got = eng.conv_forward_batch(xs, w, packing.ConvShape(10, 10, 3, 1))
    for bi in range(3):
        assert np.array_equal(got[bi], eng.conv_forward(xs[bi], w, packing.ConvShape(10, 10, 3, 1)))
    gys = rng.integers(-20, 20, size=(3, 3, 10, 10))
    gw = eng.conv_pairwise_batch(xs, gys, packing.ConvShape(10, 10, 10, 1))
    for bi in range(3):
        assert np.array_equal(gw[bi], eng.conv_pairwise(xs[bi], gys[bi], packing.ConvShape(10, 10, 10, 1)))
    # precompute mode with explicit offline for the batch job shape
    sess2 = engine.DeviceSession(params)
    eng2 = engine.DeviceSecureEngine(sess2)
    jobs = [linprot.conv_job(f"cb.b{b}", xs[b], w, packing.ConvShape(10, 10, 3, 1), eng2.ring) for b in range(3)]
    sess2.ensure_offline([eng2.batch_shape(jobs, "cb")], 1)
    assert np.array_equal(eng2.conv_forward_batch(xs, w, packing.ConvShape(10, 10, 3, 1), job_id="cb"), got)

