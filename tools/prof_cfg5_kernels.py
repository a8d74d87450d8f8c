"""Small fixed cfg5-shape workload for ncu captures of the 50-bit (N=8192, 3 x 50-bit) server kernels:
one image's conv2 weight-gradient job (4096 sites: offline per-site CCMul sums + the online step).

    python tools/prof_cfg5_kernels.py [family] [images]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2409_16675_b200 import workloads as W  # noqa: E402
from paper_2409_16675_b200.params import p8192_he_params  # noqa: E402

fam = sys.argv[1] if len(sys.argv) > 1 else "conv2_gw"
images = int(sys.argv[2]) if len(sys.argv) > 2 else 1
P = p8192_he_params()
sess = W.Session.create(P)
T = W.cfg5_tensors(images, seed=7)
gen = torch.Generator(device="cuda")
gen.manual_seed(1)
r = W.run_cfg5(sess, T, gen, group=images, families=[fam])
torch.cuda.synchronize()
ref = W.cfg5_reference_float(T)[fam]
assert torch.equal(r["outputs"][fam], ref), "mismatch"
print("ok", fam, r["offline_ms"], r["online_ms"])
