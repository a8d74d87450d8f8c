"""Fixed workload for ncu captures of the client-side encode / decode and transfer kernels:
one cfg4 batch (32 images) online step (k_pack_gather, k_decrypt_round_lazy with the extraction
epilogue) and one packed-format round trip of a cfg2a batch (k_bits_unpack / k_bits_pack)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2409_16675_b200 import workloads as W  # noqa: E402
from paper_2409_16675_b200.device import RnsContext  # noqa: E402
from paper_2409_16675_b200.params import default_he_params  # noqa: E402

P = default_he_params(4096)
sess = W.Session.create(P)
gen = torch.Generator(device="cuda")
gen.manual_seed(1)
x, w, gy = W.cfg4_tensors(32)
r = W.run_config(sess, W.cfg4_builders(P, x, w, gy), gen)
ctx = RnsContext.get(P.n, P.cipher_ring.primes, P.plain_ring.primes)
B = 4096
ct = torch.randint(0, 1 << 29, (B, 2, ctx.L, P.n), device="cuda", dtype=torch.int32)
packed = ctx.pack_bits(ct, ctx.q_bits)
back = ctx.unpack_bits(packed, ctx.q_bits, tuple(ct.shape), ct.dtype)
torch.cuda.synchronize()
assert torch.equal(back, ct)
print("ok", r["online_ms"])
