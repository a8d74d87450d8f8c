"""Launch ctb_probe_bfly_pass (k_cpmul's register pass, no exchanges / global traffic) for ncu."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2409_16675_b200 import _lib  # noqa: E402
from paper_2409_16675_b200.device import RnsContext  # noqa: E402
from paper_2409_16675_b200.params import default_he_params  # noqa: E402

P = default_he_params(4096)
ctx = RnsContext.get(P.n, P.cipher_ring.primes, P.plain_ring.primes)
lib = _lib.load()
sink = torch.zeros(1, dtype=torch.int64, device="cuda")
n = ctypes.c_uint64()
stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    assert lib.ctb_probe_bfly_pass(ctx._h, 2000, ctypes.c_void_p(sink.data_ptr()), ctypes.byref(n), stream) == 0
    e1.record()
    e1.synchronize()
    print(f"{n.value / e0.elapsed_time(e1) / 1e6:.1f} G bfly/s")
