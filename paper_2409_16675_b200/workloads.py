"""BASELINE.json configurations as batched device workloads (used by bench.py).

Each function runs a configuration end to end on one GPU with both parties
co-resident (the "channel" between client encryption and the server step is
device memory; wire serialization is measured separately in bench.py):

  cfg3  conv 1x28x28, 5 filters 5x5, stride 2 (= stride-1 job + subsample), batch 64
  cfg4  conv 3x32x32 -> 64 x 3x3 pad 1 forward + weight-gradient + input-gradient
        (the trainer's lowering, train.py:478-494), batch 32
  cfg5  linear portion of one training step at N=8192, 3 x 50-bit limbs, batch 32

Per image and job the protocol is the reference's precompute protocol
(linprot.py:387-485): offline mask products [r_x r_w] per slot from per-site
CCMul, online 2 CPMul + PPMul per site (here: one fused eval-domain call per
job batch).  Jobs of all images are concatenated block-diagonally so one
library call serves the whole batch; results are bit-identical to running the
images one by one (each image keeps its own masks and sites).
"""
from __future__ import annotations

import dataclasses
import time

import numpy as np
import torch

from . import linprot, packing
from .he import CiphertextBatch, He, KeySet
from .linprot import JobShape, LinearJob
from .ring import RingParams


def concat_jobs(jobs: list[LinearJob], job_id: str) -> tuple[LinearJob, list[JobShape]]:
    """Block-diagonal union of per-image jobs (site indices offset per image)."""
    sites, xo, wo, oo = [], 0, 0, 0
    for j in jobs:
        s = j.shape
        sites.extend((x + xo, w + wo, o + oo) for x, w, o in s.sites)
        xo, wo, oo = xo + s.n_x, wo + s.n_w, oo + s.n_out
    js = JobShape(job_id, xo, wo, oo, tuple(sites))
    x = torch.cat([j.x_plain for j in jobs])
    w = torch.cat([j.w_plain for j in jobs])
    return LinearJob(js, x, w, None, jobs[0].plain_ring), [j.shape for j in jobs]


@dataclasses.dataclass
class Session:
    """Client and server evaluators plus keys for a co-resident run."""

    client: He
    server: He
    keys: KeySet
    pks: object

    @staticmethod
    def create(params, keygen_seed: int = 1) -> "Session":
        cli, srv = He(params), He(params)
        keys = cli.keygen(keygen_seed)
        pks = srv.public_keys_from_bytes(cli.public_keys_to_bytes(keys))
        return Session(cli, srv, keys, pks)


def offline(sess: Session, job: LinearJob, gen) -> tuple[linprot.MaskBundle, CiphertextBatch]:
    """Client masks + encryptions, server per-site CCMul and slot accumulation."""
    js = job.shape
    t = sess.client.params.t
    if isinstance(gen, torch.Generator):
        r = torch.randint(0, t, (js.n_x + js.n_w, sess.client.params.n), generator=gen, device="cuda",
                          dtype=torch.int64)
    else:
        r = linprot._plain_random(sess.client, js.n_x + js.n_w, gen)
    cts = sess.client.encrypt_many(r, sess.keys, gen)
    fresh = sess.server.params.fresh_noise
    rx = CiphertextBatch(cts.data[:js.n_x], fresh, cts.backend_tag, cts._cipher)
    rw = CiphertextBatch(cts.data[js.n_x:], fresh, cts.backend_tag, cts._cipher)
    prod = linprot.attach_eval_form(sess.server, linprot._sites_ccmul_sum(sess.server, sess.pks, rx, rw, js))
    return linprot.MaskBundle(js.job_id, r[:js.n_x], r[js.n_x:]), prod


def online(sess: Session, job: LinearJob, bundle: linprot.MaskBundle, maskprod: CiphertextBatch, gen) -> torch.Tensor:
    """Client encrypt + mask, server fused linear step, client decrypt - p.  Returns [n_out, N] mod t."""
    js = job.shape
    cli, srv = sess.client, sess.server
    cx = cli.encrypt_many(job.x_plain, sess.keys, gen)
    cw = cli.encrypt_many(job.w_plain, sess.keys, gen)
    mx = linprot._plain_sub(cli, job.x_plain, bundle.r_x)
    mw = linprot._plain_sub(cli, job.w_plain, bundle.r_w)
    c_slots, p_slots = linprot.linear_online(srv, cx, cw, mx, mw, js, maskprod)
    c = cli.decrypt_values(c_slots, sess.keys)
    return linprot._plain_sub(cli, c, p_slots)


def _sync():
    torch.cuda.synchronize()


# ---------------------------------------------------------------------------------------- cfg4

def cfg4_jobs(params, images: int = 32, seed: int = 4):
    """x in [0,2^8) (B,3,32,32), w in [-2^7,2^7) (64,3,3,3), gy in [-2^7,2^7) (B,64,32,32)."""
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    x = torch.randint(0, 256, (images, 3, 32, 32), generator=g, device="cuda", dtype=torch.int64)
    w = torch.randint(-128, 128, (64, 3, 3, 3), generator=g, device="cuda", dtype=torch.int64)
    gy = torch.randint(-128, 128, (images, 64, 32, 32), generator=g, device="cuda", dtype=torch.int64)
    pr = params.plain_ring
    wrot = torch.flip(w, dims=(2, 3)).transpose(0, 1).contiguous()          # train.py:487
    fwd = [linprot.conv_job(f"fwd{b}", x[b], w, packing.ConvShape(32, 32, 3, 1), pr) for b in range(images)]
    gw = [linprot.conv_grad_w_job(f"gw{b}", x[b], gy[b], packing.ConvShape(32, 32, 32, 1), pr) for b in range(images)]
    gx = [linprot.conv_job(f"gx{b}", gy[b], wrot, packing.ConvShape(32, 32, 3, 1), pr) for b in range(images)]
    return (x, w, gy), {"fwd": fwd, "gw": gw, "gx": gx}


def run_config(sess: Session, per_image: dict, gen, check=None) -> dict:
    """Offline then online for every job family; returns timings (ms) and outputs."""
    res = {"offline_ms": 0.0, "online_ms": 0.0, "outputs": {}, "sites": 0, "ccmul": 0}
    batched = {k: concat_jobs(v, k) for k, v in per_image.items()}
    prepared = {}
    _sync()
    t0 = time.perf_counter()
    for k, (job, _) in batched.items():
        prepared[k] = offline(sess, job, gen)
        res["ccmul"] += len(job.shape.sites)
    _sync()
    res["offline_ms"] = 1e3 * (time.perf_counter() - t0)
    _sync()
    t0 = time.perf_counter()
    outs = {}
    for k, (job, _) in batched.items():
        bundle, mp = prepared[k]
        outs[k] = online(sess, job, bundle, mp, gen)
        res["sites"] += len(job.shape.sites)
    _sync()
    res["online_ms"] = 1e3 * (time.perf_counter() - t0)
    # split back per image and extract (client-side decode, outside the timed region)
    for k, (job, shapes) in batched.items():
        o, parts = 0, []
        for img_job, s in zip(per_image[k], shapes):
            parts.append(img_job.extract(outs[k][o:o + s.n_out]))
            o += s.n_out
        res["outputs"][k] = torch.stack(parts)
    return res


def conv_reference_float(x, w, pad):
    """Plain convolution on the GPU in float64 (exact at these magnitudes) -- a sanity check."""
    import torch.nn.functional as F
    return F.conv2d(x.double(), w.double(), padding=pad).round().to(torch.int64)


def signed(t: torch.Tensor, modulus: int) -> torch.Tensor:
    return packing.to_signed_tensor(t, modulus)


# ---------------------------------------------------------------------------------------- cfg5

def upsample2(g: torch.Tensor, size: int) -> torch.Tensor:
    """Zero-upsample a stride-2 output gradient onto the stride-1 grid."""
    out = torch.zeros((*g.shape[:-2], size, size), dtype=g.dtype, device=g.device)
    out[..., ::2, ::2] = g
    return out


def cfg5_tensors(images: int = 32, seed: int = 5):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)

    def r(lo, hi, *shape):
        return torch.randint(lo, hi, shape, generator=g, device="cuda", dtype=torch.int64)

    return {
        "x": r(0, 256, images, 3, 32, 32), "w1": r(-128, 128, 64, 3, 3, 3), "gy1": r(-128, 128, images, 64, 32, 32),
        "a1": r(0, 256, images, 64, 32, 32), "w2": r(-128, 128, 64, 64, 3, 3), "gy2": r(-128, 128, images, 64, 16, 16),
        "a2": r(0, 256, images, 64, 16, 16), "wfc": r(-128, 128, 10, 64 * 16 * 16), "gfc": r(-128, 128, images, 10),
    }


def cfg5_image_jobs(params, T: dict, b: int, n_chunk: int) -> dict:
    """Per image: the trainer's linear jobs (train.py:353-494 lowering) plus the stride-2 and
    FC-chunk lowerings the reference lacks; 12,733 sites at N=8192."""
    pr = params.plain_ring
    CS = packing.ConvShape
    w2rot = torch.flip(T["w2"], dims=(2, 3)).transpose(0, 1).contiguous()
    gy2u = upsample2(T["gy2"][b], 32)
    xfc = T["a2"][b].reshape(-1)
    jobs = {
        "conv1_fwd": linprot.conv_job(f"c1f{b}", T["x"][b], T["w1"], CS(32, 32, 3, 1), pr),
        "conv1_gw": linprot.conv_grad_w_job(f"c1w{b}", T["x"][b], T["gy1"][b], CS(32, 32, 32, 1), pr),
        "conv2_fwd": linprot.conv_job(f"c2f{b}", T["a1"][b], T["w2"], CS(32, 32, 3, 1), pr),
        "conv2_gx": linprot.conv_job(f"c2x{b}", gy2u, w2rot, CS(32, 32, 3, 1), pr),
        "conv2_gw": linprot.conv_grad_w_job(f"c2w{b}", T["a1"][b], gy2u, CS(32, 32, 32, 1), pr),
        "fc_gx": linprot.fc_job(f"fcx{b}", T["gfc"][b], T["wfc"].t().contiguous(), pr),
    }
    for c, lo in enumerate(range(0, xfc.numel(), n_chunk)):
        hi = lo + n_chunk
        jobs[f"fc_fwd{c}"] = linprot.fc_job(f"fcf{b}_{c}", xfc[lo:hi], T["wfc"][:, lo:hi], pr)
        jobs[f"fc_gw{c}"] = linprot.outer_job(f"fcw{b}_{c}", T["gfc"][b], xfc[lo:hi], pr)
    return jobs


WEIGHT_GRADIENT_FAMILIES = ("conv1_gw", "conv2_gw", "fc_gw0", "fc_gw1")


def run_cfg5(sess: Session, T: dict, gen, group: int = 4, families=None) -> dict:
    """Offline + online for every image (processed in groups of `group` images to bound HBM),
    outputs decoded per family; timings in ms (device-synchronised)."""
    P = sess.client.params
    images = T["x"].shape[0]
    res = {"offline_ms": {}, "online_ms": {}, "sites": {}, "outputs": {}}
    for g0 in range(0, images, group):
        per_image = [cfg5_image_jobs(P, T, b, P.n) for b in range(g0, min(images, g0 + group))]
        fams = families or list(per_image[0])
        for fam in fams:
            jobs = [pi[fam] for pi in per_image]
            job, shapes = concat_jobs(jobs, fam)
            _sync()
            t0 = time.perf_counter()
            bundle, mp = offline(sess, job, gen)
            _sync()
            t1 = time.perf_counter()
            out = online(sess, job, bundle, mp, gen)
            _sync()
            t2 = time.perf_counter()
            res["offline_ms"][fam] = res["offline_ms"].get(fam, 0.0) + 1e3 * (t1 - t0)
            res["online_ms"][fam] = res["online_ms"].get(fam, 0.0) + 1e3 * (t2 - t1)
            res["sites"][fam] = res["sites"].get(fam, 0) + len(job.shape.sites)
            o, parts = 0, []
            for img_job, s in zip(jobs, shapes):
                parts.append(img_job.extract(out[o:o + s.n_out]))
                o += s.n_out
            res["outputs"].setdefault(fam, []).extend(parts)
            del bundle, mp, out
    res["outputs"] = {k: torch.stack(v) for k, v in res["outputs"].items()}
    return res


def cfg5_reference_float(T: dict) -> dict:
    """Plain GPU float64 results of every cfg5 family (exact at these magnitudes)."""
    x, w1, gy1, a1, w2, gy2, a2, wfc, gfc = (T[k] for k in ("x", "w1", "gy1", "a1", "w2", "gy2", "a2", "wfc", "gfc"))
    B = x.shape[0]
    gy2u = upsample2(gy2, 32)
    w2rot = torch.flip(w2, dims=(2, 3)).transpose(0, 1).contiguous()
    conv = conv_reference_float
    ref = {
        "conv1_fwd": conv(x, w1, 1),
        "conv1_gw": torch.stack([conv(x[b][:, None], gy1[b][:, None], 1).transpose(0, 1) for b in range(B)]),
        "conv2_fwd": conv(a1, w2, 1),
        "conv2_gx": conv(gy2u, w2rot, 1),
        "conv2_gw": torch.stack([conv(a1[b][:, None], gy2u[b][:, None], 1).transpose(0, 1) for b in range(B)]),
        "fc_gx": (gfc.double() @ wfc.double()).round().to(torch.int64),
    }
    xf = a2.reshape(B, -1)
    n = xf.shape[1] // 2
    for c in range(2):
        sl = slice(c * n, (c + 1) * n)
        ref[f"fc_fwd{c}"] = (xf[:, sl].double() @ wfc[:, sl].double().t()).round().to(torch.int64)
        ref[f"fc_gw{c}"] = (gfc[:, :, None].double() * xf[:, None, sl].double()).round().to(torch.int64)
    return ref
