"""Time the streaming transforms (ctb_ntt_forward / inverse / mul_prepared) on a large batch."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2409_16675_b200 import _lib  # noqa: E402
from paper_2409_16675_b200.device import RnsContext, _ptr, _stream  # noqa: E402
from paper_2409_16675_b200.params import default_he_params, p8192_he_params  # noqa: E402


def run(P, npoly=8192, reps=10):
    ctx = RnsContext.get(P.n, P.cipher_ring.primes, P.plain_ring.primes)
    L, n = ctx.L, P.n
    dt = ctx.dtype()
    p = torch.tensor(P.cipher_ring.primes, dtype=torch.int64, device="cuda").view(1, L, 1)
    a = (torch.randint(0, 1 << 62, (npoly, L, n), device="cuda") % p).to(dt)
    out = torch.empty_like(a)
    key = torch.empty((1, L, n), dtype=dt, device="cuda")
    _lib.check(ctx._lib.ctb_prepare_operand(ctx._h, 0, _ptr(a[:1]), _ptr(key), 1, _stream()), "prep")
    lib, h = ctx._lib, ctx._h
    ops = {
        "fwd": lambda: lib.ctb_ntt_forward(h, 0, _ptr(a), _ptr(out), npoly, _stream()),
        "inv": lambda: lib.ctb_ntt_inverse(h, 0, _ptr(a), _ptr(out), npoly, _stream()),
        "mul_prepared": lambda: lib.ctb_mul_prepared(h, 0, _ptr(a), _ptr(key), 0, None, _ptr(out), npoly, _stream()),
    }
    for name, f in ops.items():
        for _ in range(3):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        ntts = npoly * L * (2 if name == "mul_prepared" else 1)
        print(f"N={n} L={L} {name:13s} {ms*1e3:8.1f} us  {ntts/ms/1e3:7.1f} M NTT/s  "
              f"{npoly*L*n*dt.itemsize*2/ms/1e6:7.1f} GB/s")


run(default_he_params(4096))
run(p8192_he_params(), npoly=4096)
