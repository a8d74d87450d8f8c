"""cfg5 on the GPU: linear portion of one training step at N=8192, 3 x 50-bit, with checks.

    python tools/run_cfg5.py [images] [group]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2409_16675_b200 import workloads as W  # noqa: E402
from paper_2409_16675_b200.params import p8192_he_params  # noqa: E402

images = int(sys.argv[1]) if len(sys.argv) > 1 else 1
group = int(sys.argv[2]) if len(sys.argv) > 2 else 1
P = p8192_he_params()
sess = W.Session.create(P)
gen = torch.Generator(device="cuda")
gen.manual_seed(55)
T = W.cfg5_tensors(images)
t0 = time.perf_counter()
r = W.run_cfg5(sess, T, gen, group=group)
wall = time.perf_counter() - t0
ref = W.cfg5_reference_float(T)
ok = {k: bool(torch.equal(v, ref[k])) for k, v in r["outputs"].items()}
print(json.dumps({"images": images, "wall_s": wall, "offline_ms": r["offline_ms"], "online_ms": r["online_ms"],
                  "sites": r["sites"], "exact": ok, "total_sites": sum(r["sites"].values())}, indent=1))
