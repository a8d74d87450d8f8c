"""GPU self-check of the FP64-quotient butterfly product (csrc/ntt.cuh F64Q_NE): every entry of
every 32-bit prime's quotient table, as built on the device, against exact 64-bit arithmetic for
boundary and random inputs (ctb_check_f64q).  The transforms that use it are additionally covered
bit-exactly against the oracle by test_gpu_ring.py / test_gpu_he.py."""
import ctypes

import pytest

from conftest import has_gpu
from oracle import he_ref as H
from oracle import ring_ref as R

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def _check(ctx, base, samples=4096, seed=7):
    from paper_2409_16675_b200 import _lib
    bad = ctypes.c_uint64(123)
    rc = ctx._lib.ctb_check_f64q(ctx._h, base, samples, seed, ctypes.byref(bad), None)
    assert rc == 0, ctx._lib.ctb_last_error()
    return bad.value


@pytest.mark.parametrize("n", [16, 256, 1024, 2048, 4096, 8192])
def test_quotient_tables_every_prime(n):
    from paper_2409_16675_b200 import _lib
    from paper_2409_16675_b200.device import RnsContext
    qs = R.ntt_primes(n, 30, 7)
    ctx = RnsContext.get(n, qs)
    assert _check(ctx, _lib.BASE_Q) == 0


def test_default_params_cipher_and_plain_bases():
    from paper_2409_16675_b200 import _lib
    from paper_2409_16675_b200.device import RnsContext
    P = H.default_params(4096)
    ctx = RnsContext.get(P.n, P.q_primes, P.t_primes)
    assert _check(ctx, _lib.BASE_Q, samples=1 << 16) == 0
    assert _check(ctx, _lib.BASE_T, samples=1 << 14) == 0


def test_64bit_bases_are_a_noop():
    from paper_2409_16675_b200 import _lib
    from paper_2409_16675_b200.device import RnsContext
    from paper_2409_16675_b200.params import p8192_he_params
    P = p8192_he_params()
    ctx = RnsContext.get(P.n, P.cipher_ring.primes, P.plain_ring.primes)
    assert _check(ctx, _lib.BASE_Q) == 0
