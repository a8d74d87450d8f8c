"""Chunk / slot sweep of the packed end-to-end CPMul pipeline (RnsContext.cpmul_host_packed)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2409_16675_b200.device import RnsContext  # noqa: E402
from paper_2409_16675_b200.params import default_he_params  # noqa: E402

P = default_he_params(4096)
qs = P.cipher_ring.primes
ctx = RnsContext.get(P.n, qs, P.plain_ring.primes)
B = 4096
ct = torch.empty((B, 2, len(qs), P.n), dtype=torch.int32, device="cuda")
for i, q in enumerate(qs):
    ct[:, :, i] = torch.randint(0, q, (B, 2, P.n), device="cuda").to(torch.int32)
pt = torch.randint(0, P.t, (B, P.n), device="cuda")
ctp = ctx.pack_bits(ct, ctx.q_bits).cpu().pin_memory()
ptp = ctx.pack_bits(pt, ctx.t_bits).cpu().pin_memory()
outp = torch.empty_like(ctp).pin_memory()
for chunks in (8, 16, 32, 64, 128):
    for slots in (2, 3, 4, 6):
        for _ in range(2):
            ctx.cpmul_host_packed(ctp, ptp, outp, B, chunks=chunks, slots=slots)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            ctx.cpmul_host_packed(ctp, ptp, outp, B, chunks=chunks, slots=slots)
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e) / 5
        print(f"chunks {chunks:4d} slots {slots}: {ms:7.2f} ms  {B / ms * 1e3:9.0f} CPMul/s", flush=True)
