"""A/B timing of cfg5 (linear part of a training step at N=8192, 3 x 50-bit) on `images` images
for the library CTB_LIB points at: one warm-up group, then one timed pass."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2409_16675_b200 import _lib  # noqa: E402
from paper_2409_16675_b200 import workloads as W  # noqa: E402
from paper_2409_16675_b200.params import p8192_he_params  # noqa: E402

images = int(sys.argv[1]) if len(sys.argv) > 1 else 8
P = p8192_he_params()
sess = W.Session.create(P)
gen = torch.Generator(device="cuda")
gen.manual_seed(55)
W.run_cfg5(sess, W.cfg5_tensors(4), gen, group=4)
r = W.run_cfg5(sess, W.cfg5_tensors(images), gen, group=4)
off, on = sum(r["offline_ms"].values()), sum(r["online_ms"].values())
print(f"{_lib.LIB_PATH.parent.name:8s} cfg5 x{images}: offline {off:8.1f} ms  online {on:7.1f} ms", flush=True)
