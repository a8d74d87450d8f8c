"""Kernel breakdown of the cfg4 ONLINE phase only (offline prepared outside the profiler)."""
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


def once(prof=None):
    prepared = {k: W.offline(sess, b(), gen) for k, b in builders.items()}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if prof:
        prof.__enter__()
    for k, b in builders.items():   # from the raw tensors: build, pack + mask, encrypt, server, decrypt + extract
        W.online(sess, b(), *prepared[k], gen)
    torch.cuda.synchronize()
    if prof:
        prof.__exit__(None, None, None)
    return 1e3 * (time.perf_counter() - t0)


for _ in range(2):
    print("online ms", once())
p = profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU])
print("online ms (profiled)", once(p))
ka = p.key_averages()
tot = sum(e.self_device_time_total for e in ka if e.self_device_time_total > 0) / 1e3
print(f"sum of device time {tot:.2f} ms")
print(ka.table(sort_by="self_cuda_time_total", row_limit=25, max_name_column_width=70))
