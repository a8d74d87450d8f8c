"""Full-size BASELINE configs 3-5 end to end on the GPU (client encrypt -> offline CCMul masks ->
online server step -> client decrypt/extract), decrypted outputs compared exactly with the plain
convolution / matrix products they encode (float64 on the GPU: every sum here is an integer far
below 2^53, so the rounded result is the exact integer the reference's protocol decrypts to,
test_linprot.py:102-127 / test_acceptance.py:103-191).  Seeded synthetic inputs with the configs'
shapes and value ranges."""
import pytest
import torch

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def sess4096():
    from paper_2409_16675_b200 import workloads as W
    from paper_2409_16675_b200.params import default_he_params
    P = default_he_params(4096)
    return P, W.Session.create(P)


def test_cfg3_stride2_conv_batch64(sess4096):
    """Stride 2 as the stride-1 job whose extraction keeps every other output row / column."""
    from paper_2409_16675_b200 import workloads as W
    P, sess = sess4096
    x, w = W.cfg3_tensors(64)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(11)
    r = W.run_config(sess, W.cfg3_builders(P, x, w), gen)
    out = r["outputs"]["fwd"]
    assert out.shape == (64, 5, 12, 12)
    assert torch.equal(out, W.conv_reference_float(x, w, 0)[:, :, ::2, ::2])
    assert r["sites"] == 320 and r["ccmul"] == 320


def test_cfg4_conv_fwd_bwd_batch32(sess4096):
    from paper_2409_16675_b200 import workloads as W
    P, sess = sess4096
    x, w, gy = W.cfg4_tensors(32)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(12)
    r = W.run_config(sess, W.cfg4_builders(P, x, w, gy), gen)
    assert r["sites"] == 18432 and r["ccmul"] == 18432
    assert torch.equal(r["outputs"]["fwd"], W.conv_reference_float(x, w, 1))
    ref_gw = torch.stack([W.conv_reference_float(x[b][:, None], gy[b][:, None], 1).transpose(0, 1) for b in range(32)])
    assert torch.equal(r["outputs"]["gw"], ref_gw)
    wrot = torch.flip(w, dims=(2, 3)).transpose(0, 1).contiguous()
    assert torch.equal(r["outputs"]["gx"], W.conv_reference_float(gy, wrot, 1))


def test_cfg5_training_step_linear_n8192_batch32():
    from paper_2409_16675_b200 import workloads as W
    from paper_2409_16675_b200.params import p8192_he_params
    P8 = p8192_he_params()
    sess = W.Session.create(P8)
    T = W.cfg5_tensors(32)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(13)
    r = W.run_cfg5(sess, T, gen, group=4)
    ref = W.cfg5_reference_float(T)
    assert set(r["outputs"]) == set(ref)
    for fam, v in r["outputs"].items():
        assert torch.equal(v, ref[fam]), fam
    assert sum(r["sites"][k] for k in W.WEIGHT_GRADIENT_FAMILIES) == 137856
