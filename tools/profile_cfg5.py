"""torch.profiler kernel breakdown of cfg5 (N=8192, 3 x 50-bit) for a few images."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2409_16675_b200 import workloads as W  # noqa: E402
from paper_2409_16675_b200.params import p8192_he_params  # noqa: E402

images = int(sys.argv[1]) if len(sys.argv) > 1 else 2
P = p8192_he_params()
sess = W.Session.create(P)
gen = torch.Generator(device="cuda")
gen.manual_seed(1)
T = W.cfg5_tensors(images)
W.run_cfg5(sess, W.cfg5_tensors(1, seed=9), gen, group=1)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r = W.run_cfg5(sess, T, gen, group=images)
print("offline", sum(r["offline_ms"].values()), "online", sum(r["online_ms"].values()))
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=22, max_name_column_width=70))
