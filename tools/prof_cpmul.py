"""Short fixed CPMul workload for ncu captures (cfg2a shape, 4096 ciphertexts, 3 launches)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2409_16675_b200.device import RnsContext  # noqa: E402
from paper_2409_16675_b200.params import default_he_params, p8192_he_params  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "4096"
P = default_he_params(4096) if which == "4096" else p8192_he_params()
qs = P.cipher_ring.primes
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
ctx = RnsContext.get(P.n, qs, P.plain_ring.primes)
dt = ctx.dtype()
ct = torch.empty((B, 2, len(qs), P.n), dtype=dt, device="cuda")
for i, q in enumerate(qs):
    ct[:, :, i, :] = torch.randint(0, q, (B, 2, P.n), device="cuda", dtype=torch.int64).to(dt)
pt = torch.randint(0, P.t, (B, P.n), device="cuda", dtype=torch.int64)
out = torch.empty_like(ct)
for _ in range(3):
    ctx.cpmul(ct, pt, out=out)
torch.cuda.synchronize()
print("ok", tuple(out.shape))
