"""Run a BASELINE config workload once on the GPU with timing and a float64 sanity check.

    python tools/run_cfg.py cfg4 [images]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2409_16675_b200 import workloads as W  # noqa: E402
from paper_2409_16675_b200.params import default_he_params  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
images = int(sys.argv[2]) if len(sys.argv) > 2 else 32
P = default_he_params(4096)
t0 = time.perf_counter()
sess = W.Session.create(P)
torch.cuda.synchronize()
print(f"session {time.perf_counter()-t0:.2f}s", flush=True)
gen = torch.Generator(device="cuda")
gen.manual_seed(11)
if which == "cfg4":
    x, w, gy = W.cfg4_tensors(images)
    builders = W.cfg4_builders(P, x, w, gy)
    for rep in range(2):
        r = W.run_config(sess, builders, gen)
        print(f"rep {rep}: offline {r['offline_ms']:.1f} ms ({r['ccmul']} CCMul), online {r['online_ms']:.1f} ms "
              f"(core {r['online_core_ms']:.1f} ms, {r['sites']} sites)", flush=True)
    fwd, gw, gx = (r["outputs"][k] for k in ("fwd", "gw", "gx"))
    ok_f = torch.equal(fwd, W.conv_reference_float(x, w, 1))
    ref_gw = torch.stack([W.conv_reference_float(x[b][:, None], gy[b][:, None], 1).transpose(0, 1)
                          for b in range(images)])
    ok_gw = torch.equal(gw, ref_gw)
    wrot = torch.flip(w, dims=(2, 3)).transpose(0, 1).contiguous()
    ok_gx = torch.equal(gx, W.conv_reference_float(gy, wrot, 1))
    print("fwd/gw/gx exact:", ok_f, ok_gw, ok_gx, tuple(fwd.shape), tuple(gw.shape), tuple(gx.shape))
