"""A/B timing of the cfg2a CPMul batch and the streaming transforms for the library CTB_LIB
points at (tools/ab_variants.py); prints ms per 4096-CPMul launch and an output digest so
variants can be checked for identical results."""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2409_16675_b200 import _lib  # noqa: E402
from paper_2409_16675_b200.device import RnsContext  # noqa: E402
from paper_2409_16675_b200.params import default_he_params, p8192_he_params  # noqa: E402


def timed(f, reps):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def cpmul(P, B=4096):
    qs = P.cipher_ring.primes
    ctx = RnsContext.get(P.n, qs, P.plain_ring.primes)
    dt = ctx.dtype()
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    ct = torch.empty((B, 2, len(qs), P.n), dtype=dt, device="cuda")
    for i, q in enumerate(qs):
        ct[:, :, i, :] = torch.randint(0, q, (B, 2, P.n), generator=g, device="cuda", dtype=torch.int64).to(dt)
    pt = torch.randint(0, P.t, (B, P.n), generator=g, device="cuda", dtype=torch.int64)
    out = torch.empty_like(ct)
    ms = timed(lambda: ctx.cpmul(ct, pt, out=out), 20)
    fw = ctx.ntt_forward(ct[:1024])
    ms_f = timed(lambda: ctx.ntt_forward(ct[:1024]), 20)
    dig = hashlib.sha256(out.cpu().numpy().tobytes() + fw.cpu().numpy().tobytes()).hexdigest()[:16]
    print(f"{_lib.LIB_PATH.parent.name:8s} N={P.n} cpmul {ms:7.3f} ms ({B / ms / 1e3:6.3f} M/s)  "
          f"fwd(2048 polys) {ms_f*1e3:7.1f} us  digest {dig}", flush=True)


torch.cuda.set_device(0)
cpmul(default_he_params(4096))
if len(sys.argv) > 1 and sys.argv[1] == "all":
    cpmul(p8192_he_params())
