"""cfg5 offline / online time vs image-group size (HBM bound vs batching efficiency)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2409_16675_b200 import workloads as W  # noqa: E402
from paper_2409_16675_b200.params import p8192_he_params  # noqa: E402

P = p8192_he_params()
sess = W.Session.create(P)
gen = torch.Generator(device="cuda")
gen.manual_seed(11)
T = W.cfg5_tensors(32)
for group in [int(g) for g in (sys.argv[1:] or ["4", "8"])]:
    W.run_cfg5(sess, W.cfg5_tensors(group, seed=99), gen, group=group)
    r = W.run_cfg5(sess, T, gen, group=group)
    print(f"group {group}: offline {sum(r['offline_ms'].values()):.1f} ms, online {sum(r['online_ms'].values()):.1f} ms, "
          f"peak mem {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB", flush=True)
