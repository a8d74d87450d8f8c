"""A/B: cfg4 (and cfg3) online / offline with the job families on one stream vs concurrent streams."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2409_16675_b200 import workloads as W  # noqa: E402
from paper_2409_16675_b200.params import default_he_params  # noqa: E402

P = default_he_params(4096)
sess = W.Session.create(P)
gen = torch.Generator(device="cuda")
gen.manual_seed(11)
x, w, gy = W.cfg4_tensors(32)
b4 = W.cfg4_builders(P, x, w, gy)
ref = None
for conc in (False, True, False, True):
    W.run_config(sess, b4, gen, concurrent=conc)
    runs = [W.run_config(sess, b4, gen, concurrent=conc) for _ in range(3)]
    r = min(runs, key=lambda r: r["online_ms"])
    out = {k: v.clone() for k, v in r["outputs"].items()}
    if ref is None:
        ref = out
    assert all(torch.equal(out[k], ref[k]) for k in ref), "outputs differ"
    print(f"concurrent={conc}: online {[round(q['online_ms'], 2) for q in runs]} core "
          f"{min(q['online_core_ms'] for q in runs):.2f} offline {min(q['offline_ms'] for q in runs):.2f}", flush=True)
