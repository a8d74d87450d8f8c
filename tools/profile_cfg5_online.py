"""torch.profiler kernel breakdown of ONE cfg5 family's online step for one 4-image group
(offline prepared outside the profiler).   python tools/profile_cfg5_online.py [family]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2409_16675_b200 import workloads as W  # noqa: E402
from paper_2409_16675_b200.params import p8192_he_params  # noqa: E402

fam = sys.argv[1] if len(sys.argv) > 1 else "conv2_fwd"
P = p8192_he_params()
sess = W.Session.create(P)
gen = torch.Generator(device="cuda")
gen.manual_seed(1)
T = W.cfg5_tensors(4, seed=3)
b = W.cfg5_builders(P, T, 0, 4, P.n)
for rep in range(3):
    bundle, mp = W.offline(sess, b[fam](), gen)
    torch.cuda.synchronize()
    prof = profile(activities=[ProfilerActivity.CUDA]) if rep == 2 else None
    if prof:
        prof.__enter__()
    t0 = time.perf_counter()
    W.online(sess, b[fam](), bundle, mp, gen)
    torch.cuda.synchronize()
    ms = 1e3 * (time.perf_counter() - t0)
    if prof:
        prof.__exit__(None, None, None)
    print(fam, "online ms", round(ms, 2))
print(prof.key_averages().table(sort_by="self_cuda_time_total", row_limit=16, max_name_column_width=70))
