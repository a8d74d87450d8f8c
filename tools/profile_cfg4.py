"""torch.profiler breakdown (CUDA kernels incl. libctb200 + host ops) of one cfg4 run."""
import sys
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
W.run_config(sess, builders, gen)
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    r = W.run_config(sess, builders, gen)
print("offline", r["offline_ms"], "online", r["online_ms"])
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25, max_name_column_width=60))
