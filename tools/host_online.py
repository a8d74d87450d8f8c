"""Host-side overhead of the cfg4 online phase: wall time vs device time, and a cProfile of the
Python/launch work (which host calls block on the device shows up as cumtime in sync points)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2409_16675_b200 import workloads as W  # noqa: E402
from paper_2409_16675_b200.params import default_he_params  # noqa: E402

P = default_he_params(4096)
sess = W.Session.create(P)
gen = torch.Generator(device="cuda")
gen.manual_seed(1)
x, w, gy = W.cfg4_tensors(32)
builders = W.cfg4_builders(P, x, w, gy)
prepared = {k: W.offline(sess, b(), gen) for k, b in builders.items()}


def once():
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k, b in builders.items():
        W.online(sess, b(), *prepared[k], gen)
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0)


for _ in range(3):
    print("online ms", round(once(), 3))
p = profile(activities=[ProfilerActivity.CUDA])
with p:
    once()
ka = p.key_averages()
tot = sum(e.self_device_time_total for e in ka if e.self_device_time_total > 0) / 1e3
print(f"sum of device time {tot:.2f} ms")
print(ka.table(sort_by="self_cuda_time_total", row_limit=30, max_name_column_width=60))
pr = cProfile.Profile()
pr.enable()
ms = once()
pr.disable()
print("online ms (cProfile)", round(ms, 3))
pstats.Stats(pr).sort_stats("tottime").print_stats(35)
