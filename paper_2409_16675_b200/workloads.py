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
    """Block-diagonal union of per-image jobs given as packed polynomials (site indices offset per
    image).  The batched builders (linprot.conv_job_batch & co.) build such unions directly from
    the raw tensors; this is for arbitrary job lists."""
    sites, xo, wo, oo = [], 0, 0, 0
    for j in jobs:
        arr = j.shape.sites_array().astype(np.int64)
        sites.append(arr + np.array([xo, wo, oo], dtype=np.int64))
        s = j.shape
        xo, wo, oo = xo + s.n_x, wo + s.n_w, oo + s.n_out
    js = JobShape(job_id, xo, wo, oo, np.concatenate(sites) if sites else np.zeros((0, 3)))
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


def online(sess: Session, job: LinearJob, bundle: linprot.MaskBundle, maskprod: CiphertextBatch, gen,
           decode: bool = True, centered: bool = True) -> torch.Tensor:
    """One online job, client and server co-resident (linprot.py:430-485):

      client  pack + mask      ctb_pack_gather (x, x - r_x and w, w - r_w in one kernel per side)
              encrypt          ctb_encrypt (device draws) of the packed values
      server  linear step      ctb_linear_online
      client  decrypt + decode ctb_mul_prepared_strided + ctb_decrypt_round_extract (c - p,
                               extraction and centring in the rounding kernel's epilogue)

    decode=True returns the job's centred output tensor; decode=False (or a job without a decode
    descriptor) returns the [n_out, N] mod-t polynomials decrypt(c) - p.  centered=False decodes to
    residues in [0, t) (the reference's job.extract) instead of to_signed_matrix values."""
    js = job.shape
    cli, srv = sess.client, sess.server
    mx, mw = job.masked(cli.ctx, bundle.r_x, bundle.r_w)
    cx, cw = job.encrypt_operands(cli, sess.keys, gen)
    c_slots, p_slots = linprot.linear_online(srv, cx, cw, mx, mw, js, maskprod)
    if decode and job.out is not None:
        return cli.decrypt_extract(c_slots, sess.keys, job.out, sub=p_slots, centered=centered)
    c = cli.decrypt_values(c_slots, sess.keys)
    return linprot._plain_sub(cli, c, p_slots)


def _sync():
    torch.cuda.synchronize()


# ---------------------------------------------------------------------------------------- cfg3 / cfg4

def cfg3_tensors(images: int = 64, seed: int = 3):
    """x in [0,2^8) (B,1,28,28), w in [-2^7,2^7) (5,1,5,5)."""
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    x = torch.randint(0, 256, (images, 1, 28, 28), generator=g, device="cuda", dtype=torch.int64)
    w = torch.randint(-128, 128, (5, 1, 5, 5), generator=g, device="cuda", dtype=torch.int64)
    return x, w


def cfg3_builders(params, x, w):
    """conv 1x28x28, 5 filters 5x5, stride 2: the stride-1 job with a stride-2 extraction."""
    pr = params.plain_ring
    return {"fwd": lambda: linprot.conv_job_batch("cfg3", x, w, packing.ConvShape(28, 28, 5, 0), pr, stride=2)}


def cfg4_tensors(images: int = 32, seed: int = 4):
    """x in [0,2^8) (B,3,32,32), w in [-2^7,2^7) (64,3,3,3), gy in [-2^7,2^7) (B,64,32,32)."""
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    x = torch.randint(0, 256, (images, 3, 32, 32), generator=g, device="cuda", dtype=torch.int64)
    w = torch.randint(-128, 128, (64, 3, 3, 3), generator=g, device="cuda", dtype=torch.int64)
    gy = torch.randint(-128, 128, (images, 64, 32, 32), generator=g, device="cuda", dtype=torch.int64)
    return x, w, gy


def cfg4_builders(params, x, w, gy):
    """The trainer's lowering of one conv layer's forward and backward (train.py:478-494), batched:
    fwd conv(x, w), grad-w conv_grad_w(x, gy) with the 32x32 gradient as the kernel, grad-x
    conv(gy, rot180(w)^T)."""
    pr = params.plain_ring
    wrot = torch.flip(w, dims=(2, 3)).transpose(0, 1).contiguous()          # train.py:487
    return {
        "fwd": lambda: linprot.conv_job_batch("fwd", x, w, packing.ConvShape(32, 32, 3, 1), pr),
        "gw": lambda: linprot.conv_grad_w_job_batch("gw", x, gy, packing.ConvShape(32, 32, 32, 1), pr),
        "gx": lambda: linprot.conv_job_batch("gx", gy, wrot, packing.ConvShape(32, 32, 3, 1), pr),
    }


def job_dims(js: JobShape) -> tuple[int, int, int, int]:
    """(n_x, n_w, n_out, sites) of a job: what the roofline work counts (workcount.py) need."""
    return js.n_x, js.n_w, js.n_out, len(js)


class _Concurrent:
    """Runs independent job families on their own CUDA streams (the three jobs of a conv layer's
    forward / weight-gradient / input-gradient step share no data): the host enqueues them one after
    the other, the device overlaps one job's latency-bound kernels (gathers, decryption, small
    launches) with another's transforms.  Everything before is visible to every stream, and the
    current stream waits for all of them on exit."""

    _pool: list = []   # streams are created once and reused: the caching allocator keeps a block
    #                    pool per stream, so fresh streams per call would re-allocate every buffer

    def __init__(self, n: int, enabled: bool = True):
        self.enabled = enabled and n > 1
        if self.enabled:
            while len(_Concurrent._pool) < n:
                _Concurrent._pool.append(torch.cuda.Stream())
        self.streams = _Concurrent._pool[:n] if self.enabled else []

    def __enter__(self):
        if self.enabled:
            ev = torch.cuda.Event()
            ev.record()
            for s in self.streams:
                s.wait_event(ev)
        return self

    def stream(self, i: int):
        return torch.cuda.stream(self.streams[i]) if self.enabled else _null()

    def __exit__(self, *a):
        cur = torch.cuda.current_stream()
        for s in self.streams:
            cur.wait_stream(s)


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def run_config(sess: Session, builders: dict, gen, concurrent: bool = True) -> dict:
    """Offline (the families' CCMul sums concurrently on their own streams when `concurrent`:
    measured 54.2 -> 50.9 ms for cfg4; the online phase measured slower that way -- its persistent
    transform kernels fill every SM -- and stays on one stream), then the online phase twice over
    every job family:

      online_ms        the whole client + server step from the raw tensors: job build (cached
                       descriptors), pack + mask, encrypt, server step, decrypt + extract + centre
      online_core_ms   the same without encode / decode: operands packed and masked before the
                       timer, the result left as [n_out, N] mod-t polynomials (decrypt(c) - p)
    Returns timings (ms, host-timed around device-synchronised regions) and the decoded outputs."""
    res = {"offline_ms": 0.0, "online_ms": 0.0, "online_core_ms": 0.0, "outputs": {}, "sites": 0, "ccmul": 0}
    shapes = {k: b() for k, b in builders.items()}
    res["shapes"] = {k: job_dims(j.shape) for k, j in shapes.items()}
    prepared = {}
    _sync()
    t0 = time.perf_counter()
    with _Concurrent(len(shapes), concurrent) as cc:
        for i, (k, job) in enumerate(shapes.items()):
            with cc.stream(i):
                prepared[k] = offline(sess, job, gen)
            res["ccmul"] += len(job.shape)
    _sync()
    res["offline_ms"] = 1e3 * (time.perf_counter() - t0)
    # online, encode/decode included
    _sync()
    t0 = time.perf_counter()
    with _Concurrent(len(builders), concurrent) as cc:
        for i, (k, build) in enumerate(builders.items()):
            # one family after the other, each on the stream its offline step used (its freed blocks
            # are in that stream's allocator pool); the next waits for it
            with cc.stream(i):
                job = build()
                bundle, mp = prepared[k]
                res["outputs"][k] = online(sess, job, bundle, mp, gen)
                done = torch.cuda.Event()
                done.record()
            if cc.enabled and i + 1 < len(cc.streams):
                cc.streams[i + 1].wait_event(done)
            res["sites"] += len(job.shape)
    _sync()
    res["online_ms"] = 1e3 * (time.perf_counter() - t0)
    # online core: pre-packed, pre-masked operands; no extraction (reuses the masks above: timing
    # only, the outputs are discarded)
    pre = {}
    for k, build in builders.items():
        job = build()
        bundle, _ = prepared[k]
        mx, mw = job.masked(sess.client.ctx, bundle.r_x, bundle.r_w)
        pre[k] = (job, mx, mw)
    _sync()
    t0 = time.perf_counter()
    for k, (job, mx, mw) in pre.items():
        cli, srv = sess.client, sess.server
        cx = cli.encrypt_many(job.x_plain, sess.keys, gen)
        cw = cli.encrypt_many(job.w_plain, sess.keys, gen)
        c_slots, p_slots = linprot.linear_online(srv, cx, cw, mx, mw, job.shape, prepared[k][1])
        linprot._plain_sub(cli, cli.decrypt_values(c_slots, sess.keys), p_slots)
    _sync()
    res["online_core_ms"] = 1e3 * (time.perf_counter() - t0)
    return res


def conv_reference_float(x, w, pad):
    """Plain convolution on the GPU in float64 (exact at these magnitudes) -- a sanity check."""
    import torch.nn.functional as F
    return F.conv2d(x.double(), w.double(), padding=pad).round().to(torch.int64)


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


def cfg5_builders(params, T: dict, lo: int, hi: int, n_chunk: int) -> dict:
    """Images lo..hi-1 of the trainer's linear jobs (train.py:353-494 lowering) batched per family,
    plus the stride-2 and FC-chunk lowerings the reference lacks; 12,733 sites per
    image at N=8192.  conv2's stride-2 forward keeps only the strided outputs in its extraction."""
    pr = params.plain_ring
    CS = packing.ConvShape
    sl = slice(lo, hi)
    w2rot = torch.flip(T["w2"], dims=(2, 3)).transpose(0, 1).contiguous()
    gy2u = upsample2(T["gy2"][sl], 32)
    xfc = T["a2"][sl].reshape(hi - lo, -1)
    b = {
        "conv1_fwd": lambda: linprot.conv_job_batch("c1f", T["x"][sl], T["w1"], CS(32, 32, 3, 1), pr),
        "conv1_gw": lambda: linprot.conv_grad_w_job_batch("c1w", T["x"][sl], T["gy1"][sl], CS(32, 32, 32, 1), pr),
        "conv2_fwd": lambda: linprot.conv_job_batch("c2f", T["a1"][sl], T["w2"], CS(32, 32, 3, 1), pr, stride=2),
        "conv2_gx": lambda: linprot.conv_job_batch("c2x", gy2u, w2rot, CS(32, 32, 3, 1), pr),
        "conv2_gw": lambda: linprot.conv_grad_w_job_batch("c2w", T["a1"][sl], gy2u, CS(32, 32, 32, 1), pr),
        "fc_gx": lambda: linprot.fc_job_batch("fcx", T["gfc"][sl], T["wfc"].t().contiguous(), pr),
    }
    for c, c0 in enumerate(range(0, xfc.shape[1], n_chunk)):
        xs = xfc[:, c0:c0 + n_chunk].contiguous()       # the client's inputs, chunked once
        ws = T["wfc"][:, c0:c0 + n_chunk].contiguous()
        b[f"fc_fwd{c}"] = (lambda xs=xs, ws=ws: linprot.fc_job_batch("fcf", xs, ws, pr))
        b[f"fc_gw{c}"] = (lambda xs=xs: linprot.outer_job_batch("fcw", T["gfc"][sl], xs, pr))
    return b


WEIGHT_GRADIENT_FAMILIES = ("conv1_gw", "conv2_gw", "fc_gw0", "fc_gw1")


def run_cfg5(sess: Session, T: dict, gen, group: int = 4, families=None, concurrent: bool = True) -> dict:
    """Offline + online for every image (processed in groups of `group` images to bound HBM),
    outputs decoded per family (centred); timings in ms (device-synchronised).  The online time
    includes encode (pack + mask) and decode (extraction in the decrypt epilogue).

    concurrent=True runs a group's offline jobs (all families) on their own streams at once and
    reports the offline time per group ("offline_ms" then has a single "all" entry); False runs
    family by family and reports each.  The online jobs run family by family either way."""
    P = sess.client.params
    images = T["x"].shape[0]
    res = {"offline_ms": {}, "online_ms": {}, "sites": {}, "outputs": {}, "shapes": {}}
    for g0 in range(0, images, group):
        builders = cfg5_builders(P, T, g0, min(images, g0 + group), P.n)
        fams = families or list(builders)
        shape_jobs = {fam: builders[fam]() for fam in fams}
        prepared = {}
        if concurrent:
            _sync()
            t0 = time.perf_counter()
            with _Concurrent(len(fams), True) as cc:
                for i, fam in enumerate(fams):
                    with cc.stream(i):
                        prepared[fam] = offline(sess, shape_jobs[fam], gen)
            _sync()
            res["offline_ms"]["all"] = res["offline_ms"].get("all", 0.0) + 1e3 * (time.perf_counter() - t0)
        for i, fam in enumerate(fams):
            shape_job = shape_jobs[fam]
            _sync()
            t0 = time.perf_counter()
            if not concurrent:
                prepared[fam] = offline(sess, shape_job, gen)
                _sync()
            t1 = time.perf_counter()
            bundle, mp = prepared.pop(fam)
            # (concurrent: on the family's own stream, one family at a time, so the online step
            # reuses the blocks its offline step freed in that stream's allocator pool)
            with _Concurrent(len(fams), concurrent) as cc, cc.stream(i):
                out = online(sess, builders[fam](), bundle, mp, gen)
            _sync()
            t2 = time.perf_counter()
            if not concurrent:
                res["offline_ms"][fam] = res["offline_ms"].get(fam, 0.0) + 1e3 * (t1 - t0)
            res["online_ms"][fam] = res["online_ms"].get(fam, 0.0) + 1e3 * (t2 - t1)
            res.setdefault("online_ms_calls", {}).setdefault(fam, []).append(round(1e3 * (t2 - t1), 2))
            res["sites"][fam] = res["sites"].get(fam, 0) + len(shape_job.shape)
            prev = res["shapes"].get(fam, (0, 0, 0, 0))
            res["shapes"][fam] = tuple(a + b for a, b in zip(prev, job_dims(shape_job.shape)))
            res["outputs"].setdefault(fam, []).append(out)
            del bundle, mp, out
        del shape_jobs, prepared
    res["outputs"] = {k: torch.cat(v) for k, v in res["outputs"].items()}
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
        "conv2_fwd": conv(a1, w2, 1)[:, :, ::2, ::2],
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
