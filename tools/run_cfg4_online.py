"""One cfg4 run (32 images) for profiling the online kernels under ncu."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2409_16675_b200 import workloads as W  # noqa: E402
from paper_2409_16675_b200.params import default_he_params  # noqa: E402

P = default_he_params(4096)
sess = W.Session.create(P)
gen = torch.Generator(device="cuda")
gen.manual_seed(1)
x, w, gy = W.cfg4_tensors(int(sys.argv[1]) if len(sys.argv) > 1 else 32)
r = W.run_config(sess, W.cfg4_builders(P, x, w, gy), gen)
print("offline", r["offline_ms"], "online", r["online_ms"])
