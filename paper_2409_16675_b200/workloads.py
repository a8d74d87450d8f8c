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
    prod = linprot._sites_ccmul_sum(sess.server, sess.pks, rx, rw, js)
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
    dec = cli.decrypt_many(c_slots, sess.keys)
    c = torch.stack([d.data for d in dec])
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
