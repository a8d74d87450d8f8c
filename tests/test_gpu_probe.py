"""Roofline probes of the C ABI (bench.py's denominators): they launch, count what they say they
count, and reject contexts they are not defined for."""
import ctypes

import pytest

pytestmark = pytest.mark.gpu


def _call(fn, *args):
    import torch
    sink = torch.zeros(1, dtype=torch.int64, device="cuda")
    n = ctypes.c_uint64()
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    rc = fn(*args, ctypes.c_void_p(sink.data_ptr()), ctypes.byref(n), stream)
    torch.cuda.synchronize()
    return rc, n.value, int(sink.item())


def test_probe_counts_and_sink_untouched():
    import torch
    from paper_2409_16675_b200 import _lib
    from paper_2409_16675_b200.device import RnsContext
    from paper_2409_16675_b200.params import default_he_params, p8192_he_params
    lib = _lib.load()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for fn, args in ((lib.ctb_probe_modmul_mix, (3, 10)), (lib.ctb_probe_modmul_mix_splice, (3, 10)),
                     (lib.ctb_probe_modmul_mix, (8, 10)), (lib.ctb_probe_modmul_mix_splice, (0, 10))):
        rc, n, sink = _call(fn, *args)
        assert rc == 0 and n == sms * 8 * 256 * 8 * 10 and sink == 0
    assert _call(lib.ctb_probe_modmul_mix, 5, 10)[0] != 0          # only 0, 3 or 8 of 8 chains
    P = default_he_params(4096)
    ctx = RnsContext.get(P.n, P.cipher_ring.primes, P.plain_ring.primes)
    rc, n, sink = _call(lib.ctb_probe_bfly_pass, ctx._h, 7)
    assert rc == 0 and n == sms * 1024 * 32 * 7 and sink == 0
    P8 = p8192_he_params()
    ctx8 = RnsContext.get(P8.n, P8.cipher_ring.primes, P8.plain_ring.primes)
    rc, _, _ = _call(lib.ctb_probe_bfly_pass, ctx8._h, 7)          # N = 8192 / 64-bit limbs: not defined
    assert rc != 0 and b"4096" in lib.ctb_last_error()
