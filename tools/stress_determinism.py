"""Race detector by repetition: the relaxed exchange guards (ntt.cuh Exchanger RELAX) of k_cpmul and
k_encrypt are correct by an ordering argument; a missed hazard would show as run-to-run differences.
Runs each kernel `reps` times on a full-size batch and requires bit-identical outputs every time
(and the CPMul digest the oracle-checked tests pin)."""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2409_16675_b200.device import RnsContext  # noqa: E402
from paper_2409_16675_b200.params import default_he_params  # noqa: E402
from paper_2409_16675_b200 import he as HE  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
P = default_he_params(4096)
qs = P.cipher_ring.primes
ctx = RnsContext.get(P.n, qs, P.plain_ring.primes)
g = torch.Generator(device="cuda")
g.manual_seed(5)
B = 4096
ct = torch.empty((B, 2, len(qs), P.n), dtype=ctx.dtype(), device="cuda")
for i, q in enumerate(qs):
    ct[:, :, i, :] = torch.randint(0, q, (B, 2, P.n), generator=g, device="cuda", dtype=torch.int64).to(ctx.dtype())
pt = torch.randint(0, P.t, (B, P.n), generator=g, device="cuda", dtype=torch.int64)
first = ctx.cpmul(ct, pt).clone()
bad = 0
for _ in range(reps):
    bad += int(not torch.equal(ctx.cpmul(ct, pt), first))
print("cpmul", reps, "repeats, mismatches:", bad, hashlib.sha256(first.cpu().numpy().tobytes()).hexdigest()[:16])

he = HE.He(P)
keys = he.keygen(1)
m = torch.randint(0, P.t, (2048, P.n), generator=g, device="cuda", dtype=torch.int64)
outs = []
for r in range(reps):
    gg = torch.Generator(device="cuda")
    gg.manual_seed(77)
    c = he.encrypt_many(m, keys, gg)
    outs.append(c.data if hasattr(c, "data") else c)
ebad = sum(int(not torch.equal(o, outs[0])) for o in outs[1:])
print("encrypt", reps, "repeats, mismatches:", ebad)
sys.exit(1 if bad or ebad else 0)
