"""CPU tests of the host-side logic of the device path: packing plans, job
sites and their wire format, blob framing, channel framing.  No GPU needed."""
import hashlib
import json
import struct

import numpy as np
import pytest

from paper_2409_16675_b200 import channel, packing, wire
from paper_2409_16675_b200.linprot import JobShape
from paper_2409_16675_b200.params import default_he_params


def test_choose_tiles_golden(golden):
    # reference tests/test_packing.py:169-170
    assert packing.choose_tiles(packing.ConvShape(64, 64, 5, 4), 4096) == (56, 64)
    assert list(packing.choose_tiles(packing.ConvShape(64, 64, 5, 4), 4096)) == \
        golden["packing"]["choose_tiles_64_64_5_4_4096"]


def test_plans_match_reference(golden):
    g = golden["packing"]
    assert packing.plan_correlated(packing.ConvShape(28, 28, 5, 0), 4096).row_stride == g["cfg3_plan"]
    assert packing.plan_correlated(packing.ConvShape(32, 32, 3, 1), 4096).row_stride == g["cfg4_plan"]
    p = packing.plan_correlated(packing.ConvShape(32, 32, 32, 1), 4096)
    assert [p.row_stride, p.num_tiles] == g["cfg4_gw_plan"]


def test_toy_degrees():
    # reference tests/test_packing.py:24-37: input degrees 0,1,3,4 and kernel 4,3,1,0 at 2x2/2x2 pad 1
    plan = packing.plan_correlated(packing.ConvShape(2, 2, 2, 1), 64)
    t, d, s = packing.input_index_map(plan)
    assert sorted(d.tolist()) == [0, 1, 3, 4]
    assert packing.kernel_degrees(plan).tolist() == [4, 3, 1, 0]


def test_feasibility_and_tiling_exhaustive_minimum():
    shape = packing.ConvShape(40, 40, 3, 1)
    n = 512
    hw, ww = packing.choose_tiles(shape, n)
    best = packing.tile_count(shape, hw, ww)
    for a in range(3, 41):
        for b in range(3, 41):
            if packing.window_feasible(shape, a, b, n):
                assert packing.tile_count(shape, a, b) >= best
    plan = packing.plan_correlated(shape, n)
    assert plan.degree_bound <= n - 1
    # every output entry is owned exactly once after the crop
    _, _, dst = packing.output_index_map(plan)
    assert sorted(dst.tolist()) == list(range(shape.out_height * shape.out_width))


def test_jobshape_wire_roundtrip_and_cfg4_sites(golden):
    js = JobShape("conv1", 3, 192, 64, tuple((c, co * 3 + c, co) for co in range(64) for c in range(3)))
    assert JobShape.from_bytes(js.to_bytes()) == js
    assert [js.n_x, js.n_w, js.n_out, len(js.sites)] == golden["jobs"]["cfg4_fwd"]
    sites = [list(s) for s in js.sites]
    assert hashlib.sha256(json.dumps(sites).encode()).hexdigest() == golden["jobs"]["cfg4_fwd_sites_digest"]


def test_wire_blobs_match_reference_layout():
    blobs = [b"pre", b"", b"x" * 70000]
    enc = wire.encode_blobs(blobs)
    ref = struct.pack("<I", 3) + b"".join(struct.pack("<I", len(b)) + b for b in blobs)
    assert enc == ref
    dec, off = wire.decode_blobs(enc)
    assert dec == blobs and off == len(enc)


def test_channel_framing_and_phase_checks():
    c, s = channel.inproc_pair(capture=True, timeout=2.0)
    c.send(channel.PHASE_ONLINE, b"abc")
    assert s.recv(channel.PHASE_ONLINE) == b"abc"
    s.send(channel.PHASE_SETUP, b"z")
    with pytest.raises(channel.PhaseMismatchError):
        c.recv(channel.PHASE_ONLINE)
    rep = c.stats.report()
    assert rep["bytes_client_to_server"] == 8 and rep["bytes_server_to_client"] == 6 and rep["rounds"] == 2
    assert bytes(c.stats.transcript[channel.CLIENT]) == struct.pack("<BI", 2, 3) + b"abc"


def test_params_and_noise_algebra(golden):
    P = default_he_params(4096)
    assert list(P.cipher_ring.primes) == golden["p4096"]["q_primes"]
    assert P.noise_budget.bit_length() == golden["p4096"]["noise_budget_bits"]
    with pytest.raises(ValueError):
        from paper_2409_16675_b200.params import RingParams
        RingParams(4, 15, primes=(3, 5))


def test_trainer_fixture_matches_plain_oracle():
    """The recorded reference PlainEngine outputs agree with the plain oracle (fixture sanity)."""
    from pathlib import Path
    from oracle.plainconv import conv2d_multi
    store = dict(np.load(Path(__file__).parent / "golden" / "trainer_calls.npz"))
    seen = set()
    for tag in ("toy", "bn"):
        for ci in range(int(store[f"{tag}.ncalls"])):
            pre = f"{tag}.call{ci:03d}"
            m, a, b, out = str(store[f"{pre}.method"]), store[f"{pre}.a"], store[f"{pre}.b"], store[f"{pre}.out"]
            seen.add(m)
            if m == "conv_forward":
                exp = conv2d_multi(a, b, int(store[f"{pre}.shape"][3]))
            elif m == "conv_pairwise":
                pad = int(store[f"{pre}.shape"][3])
                exp = np.stack([conv2d_multi(a[ci:ci + 1], b[:, None], pad) for ci in range(a.shape[0])], axis=1)
            elif m == "fc":
                exp = a @ b
            elif m == "outer":
                exp = np.outer(a, b)
            else:
                exp = a * int(b)
            assert np.array_equal(exp, out), (tag, ci, m)
    assert seen == {"conv_forward", "conv_pairwise", "fc", "outer", "affine"}


def test_packing_error_behaviour():
    """Reference tests/test_packing.py:99-103 (wrap detection) and :192-196 (infeasible
    budget): the same exception classes surface from the device-path packer."""
    import torch
    from paper_2409_16675_b200.params import RingParams
    h = 4
    tiny = h * (2 * h - 1) + h - 1
    with pytest.raises(packing.InfeasibleWindowError):
        packing.choose_tiles(packing.ConvShape(8, 8, h, 0), tiny)
    with pytest.raises(packing.PackingError):
        shape = packing.ConvShape(7, 7, 3, 2)
        plan = packing.plan_correlated(shape, 256, window=(7, 7))
        ring64 = RingParams(64, 17)
        packing.pack_input_batch(torch.ones((1, 7, 7), dtype=torch.int64), plan, ring64)
    P = default_he_params(4096)
    plan = packing.plan_correlated(packing.ConvShape(8, 8, 3, 1), 4096)
    with pytest.raises(packing.PackingError):  # wrong input extent
        packing.pack_input_batch(torch.ones((1, 9, 8), dtype=torch.int64), plan, P.plain_ring)
    with pytest.raises(packing.PackingError):  # wrong kernel extent
        packing.pack_kernel_batch(torch.ones((1, 2, 2), dtype=torch.int64), plan, P.plain_ring)
    with pytest.raises(packing.PackingError):  # fc input wider than the ring (packing.py:557-558)
        packing.pack_fc_input_batch(torch.ones((1, 4097), dtype=torch.int64), P.plain_ring)
