"""Sweep RnsContext.cpmul_host chunking (cfg2a e2e: pinned host buffers, H2D / CPMul / D2H)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2409_16675_b200.device import RnsContext  # noqa: E402
from paper_2409_16675_b200.params import default_he_params  # noqa: E402

P = default_he_params(4096)
ctx = RnsContext.get(P.n, P.cipher_ring.primes, P.plain_ring.primes)
B, L, n = 4096, ctx.L, P.n
p = torch.tensor(P.cipher_ring.primes, dtype=torch.int64).view(1, 1, L, 1)
ct_h = (torch.randint(0, 1 << 62, (B, 2, L, n)) % p).to(torch.int32).pin_memory()
pt_h = torch.randint(0, P.t, (B, n), dtype=torch.int64).pin_memory()
out_h = torch.empty_like(ct_h).pin_memory()
h2d = ct_h.numel() * 4 + pt_h.numel() * 8
for chunks, slots in [(8, 3), (16, 3), (32, 3), (32, 4), (64, 4), (128, 4)]:
    for _ in range(2):
        ctx.cpmul_host(ct_h, pt_h, out_h, chunks=chunks, slots=slots)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        ctx.cpmul_host(ct_h, pt_h, out_h, chunks=chunks, slots=slots)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"chunks {chunks:4d} slots {slots}: {ms:7.2f} ms/step  {B/ms*1e3:9.0f} CPMul/s  "
          f"H2D {h2d/ms/1e6:5.1f} GB/s")
# raw copy bandwidth
d = torch.empty_like(ct_h, device="cuda")
d2 = torch.empty_like(ct_h, device="cuda")
for name, f in [("H2D", lambda: d.copy_(ct_h, non_blocking=True)), ("D2H", lambda: out_h.copy_(d, non_blocking=True))]:
    f(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); f(); f(); e.record(); torch.cuda.synchronize()
    print(name, f"{2*ct_h.numel()*4/s.elapsed_time(e)/1e6:.1f} GB/s")
# both directions at once on two streams
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
with torch.cuda.stream(sa):
    d.copy_(ct_h, non_blocking=True)
with torch.cuda.stream(sb):
    out_h.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(sa); torch.cuda.current_stream().wait_stream(sb)
e.record(); torch.cuda.synchronize()
print("bidir", f"{2*ct_h.numel()*4/s.elapsed_time(e)/1e6:.1f} GB/s total")
