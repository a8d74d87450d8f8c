"""A/B timing of the cfg4 workload (batch 32 conv fwd + grad-w + grad-x, precompute protocol) for
the library CTB_LIB points at: one warm-up run, then the best of three (offline / online ms)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2409_16675_b200 import _lib  # noqa: E402
from paper_2409_16675_b200 import workloads as W  # noqa: E402
from paper_2409_16675_b200.params import default_he_params  # noqa: E402

P = default_he_params(4096)
sess = W.Session.create(P)
gen = torch.Generator(device="cuda")
gen.manual_seed(1)
x, w, gy = W.cfg4_tensors(32)
best = None
for i in range(4):
    r = W.run_config(sess, W.cfg4_builders(P, x, w, gy), gen)
    if i:
        best = (min(best[0], r["offline_ms"]), min(best[1], r["online_ms"])) if best else (r["offline_ms"], r["online_ms"])
print(f"{_lib.LIB_PATH.parent.name:8s} cfg4 offline {best[0]:7.2f} ms  online {best[1]:6.2f} ms", flush=True)
