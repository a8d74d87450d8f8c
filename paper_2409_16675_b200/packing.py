"""Correlated tensor <-> polynomial packing (mirror of privtrain.packing, correlated scheme).

Input entry (i, j) of a window starting at (r0, c0) goes to degree
(i - r0) * O + (j - c0) with row stride O = max(window) + h - 1, kernel entry
(i, j) to degree (h-1-i) * O + (h-1-j); every product coefficient at degree
u * O + v is then an output of the full-padding convolution
(packing.py:11-16, 407-509 in the reference).  Window selection is the
reference's exhaustive minimum-tile-count search with the same tie-break
(packing.py:225-260), so plans -- and therefore sites and ciphertexts -- are
identical.  Plans are value-independent and cached per (shape, degree).

The device path packs and extracts whole batches with one hand-written gather /
scatter kernel each (csrc/pack.cu; the extraction can also run as the decrypt
epilogue, ctb_decrypt_round_extract), driven by per-plan degree maps
(`Gather` / `Scatter` descriptors); the per-polynomial functions keep the
reference's signatures and return device RingElems.
The row-major "baseline" scheme and the analytic count report are
reference-side experiments outside the hot path.
"""
from __future__ import annotations

import dataclasses
import functools
import math

import numpy as np
import torch

from .ring import RingElem, RingParams

SCHEME_BASELINE = "baseline"
SCHEME_CORRELATED = "correlated"


class PackingError(Exception):
    """Base error for packing."""


class PartitionError(PackingError):
    """A requested window does not fit the degree budget."""


class InfeasibleWindowError(PackingError):
    """No window satisfies the partition constraints for this budget."""


class PackingOverflowError(PackingError):
    """Used degrees would wrap around x^n + 1."""


@dataclasses.dataclass(frozen=True)
class ConvShape:
    """Stride-1 square-kernel convolution geometry (packing.py:58-102)."""

    height: int
    width: int
    kernel: int
    pad: int = 0

    def __post_init__(self):
        if self.kernel < 1:
            raise ValueError("kernel side must be >= 1")
        if self.height < self.kernel or self.width < self.kernel:
            raise ValueError("input must be at least kernel-sized; pad first")
        if not 0 <= self.pad <= self.kernel - 1:
            raise ValueError("pad must lie in [0, kernel-1]")

    @property
    def stride_base(self) -> int:
        return max(self.width, self.height) + self.kernel - 1

    @property
    def out_height(self) -> int:
        return self.height + 2 * self.pad - self.kernel + 1

    @property
    def out_width(self) -> int:
        return self.width + 2 * self.pad - self.kernel + 1

    @property
    def full_out_height(self) -> int:
        return self.height + self.kernel - 1

    @property
    def full_out_width(self) -> int:
        return self.width + self.kernel - 1

    @property
    def padded_height(self) -> int:
        return self.height + 2 * self.pad

    @property
    def padded_width(self) -> int:
        return self.width + 2 * self.pad


@dataclasses.dataclass(frozen=True)
class Tile:
    index: int
    row0: int
    col0: int
    rows: int
    cols: int


@dataclasses.dataclass(frozen=True)
class PackingPlan:
    scheme: str
    shape: ConvShape
    n: int
    window: tuple[int, int]
    row_stride: int
    tiles: tuple[Tile, ...]
    owned: tuple[tuple[int, int, int, int], ...]
    degree_bound: int

    @property
    def num_tiles(self) -> int:
        return len(self.tiles)


# ------------------------------------------------------------------------- window selection

def _product_degree(hw: int, ww: int, h: int) -> int:
    stride = max(ww, hw) + h - 1
    return (hw + h - 2) * stride + (ww + h - 2)


def window_feasible(shape: ConvShape, hw: int, ww: int, n: int) -> bool:
    h = shape.kernel
    if not (h <= hw <= shape.height and h <= ww <= shape.width):
        return False
    stride = max(ww, hw) + h - 1
    return ww + hw * stride <= n and _product_degree(hw, ww, h) <= n - 1


def tile_count(shape: ConvShape, hw: int, ww: int) -> int:
    h = shape.kernel
    nr = math.ceil((shape.height - h + 1) / (hw - h + 1)) if hw > h - 1 else 0
    nc = math.ceil((shape.width - h + 1) / (ww - h + 1)) if ww > h - 1 else 0
    return nr * nc


@functools.lru_cache(maxsize=1024)
def choose_tiles(shape: ConvShape, n: int) -> tuple[int, int]:
    """Minimum tile count; ties prefer the larger area, then the taller window."""
    candidates = [
        ((tile_count(shape, hw, ww), -hw * ww, -hw), (hw, ww))
        for hw in range(shape.kernel, shape.height + 1)
        for ww in range(shape.kernel, shape.width + 1)
        if window_feasible(shape, hw, ww, n)
    ]
    if not candidates:
        raise InfeasibleWindowError(f"no feasible window for kernel {shape.kernel} within degree budget {n}")
    return min(candidates)[1]


def _starts(extent: int, window: int, step: int) -> list[int]:
    if window >= extent:
        return [0]
    out = list(range(0, extent - window, step))
    if not out or out[-1] != extent - window:
        out.append(extent - window)
    return list(dict.fromkeys(out))


def _ownership(starts: list[int], window: int, kernel: int, extent_out: int) -> list[tuple[int, int]]:
    spans, prev = [], 0
    last = len(starts) - 1
    for k, p0 in enumerate(starts):
        lo = 0 if k == 0 else max(p0 + kernel - 1, prev)
        hi = max(extent_out if k == last else p0 + window, lo)
        spans.append((lo, hi))
        prev = hi
    return spans


@functools.lru_cache(maxsize=1024)
def plan_correlated(shape: ConvShape, n: int, window: tuple[int, int] | None = None) -> PackingPlan:
    h = shape.kernel
    hw, ww = window if window is not None else choose_tiles(shape, n)
    if not window_feasible(shape, hw, ww, n):
        raise PartitionError(f"window {hw}x{ww} does not fit budget {n} for kernel {h} (re-tile)")
    rows = _starts(shape.height, hw, hw - h + 1)
    cols = _starts(shape.width, ww, ww - h + 1)
    row_own = _ownership(rows, hw, h, shape.full_out_height)
    col_own = _ownership(cols, ww, h, shape.full_out_width)
    tiles, owned = [], []
    for a, r0 in enumerate(rows):
        for b, c0 in enumerate(cols):
            tiles.append(Tile(len(tiles), r0, c0, hw, ww))
            owned.append(row_own[a] + col_own[b])
    return PackingPlan(SCHEME_CORRELATED, shape, n, (hw, ww), max(ww, hw) + h - 1, tuple(tiles), tuple(owned),
                       _product_degree(hw, ww, h))


def _check_plan(plan: PackingPlan, params: RingParams):
    if plan.scheme != SCHEME_CORRELATED:
        raise PackingError(f"plan is for scheme {plan.scheme!r}, not {SCHEME_CORRELATED!r}")
    if plan.n > params.n:
        raise PackingError("plan degree budget exceeds the ring degree")
    if plan.degree_bound >= params.n:
        raise PackingOverflowError(f"plan needs degree {plan.degree_bound}, ring has {params.n}")


# ------------------------------------------------------------------------- index maps

def input_index_map(plan: PackingPlan) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(tile id, degree, flat source index) of every packed input entry."""
    sh, O = plan.shape, plan.row_stride
    t_ids, degs, srcs = [], [], []
    for t in plan.tiles:
        ii, jj = np.meshgrid(np.arange(t.rows), np.arange(t.cols), indexing="ij")
        t_ids.append(np.full(ii.size, t.index))
        degs.append((ii * O + jj).ravel())
        srcs.append(((ii + t.row0) * sh.width + (jj + t.col0)).ravel())
    return np.concatenate(t_ids), np.concatenate(degs), np.concatenate(srcs)


def kernel_degrees(plan: PackingPlan) -> np.ndarray:
    h, O = plan.shape.kernel, plan.row_stride
    r = h - 1 - np.arange(h)
    return (r[:, None] * O + r[None, :]).ravel()


def output_index_map(plan: PackingPlan) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(tile id, degree, flat index into the cropped output) for every output entry."""
    sh, O = plan.shape, plan.row_stride
    crop = sh.kernel - 1 - sh.pad
    out_w = sh.out_width
    t_ids, degs, dsts = [], [], []
    for t, (u0, u1, v0, v1) in zip(plan.tiles, plan.owned):
        if u1 <= u0 or v1 <= v0:
            continue
        uu, vv = np.meshgrid(np.arange(u0, u1), np.arange(v0, v1), indexing="ij")
        keep = (uu >= crop) & (uu < crop + sh.out_height) & (vv >= crop) & (vv < crop + out_w)
        uu, vv = uu[keep], vv[keep]
        t_ids.append(np.full(uu.size, t.index))
        degs.append((uu - t.row0) * O + (vv - t.col0))
        dsts.append((uu - crop) * out_w + (vv - crop))
    return np.concatenate(t_ids), np.concatenate(degs), np.concatenate(dsts)


# ------------------------------------------------------------------------- device gather / scatter descriptors
#
# Encoding and decoding run as hand-written kernels (csrc/pack.cu, ctb_pack_gather / ctb_plain_scatter,
# and the decrypt epilogue ctb_decrypt_round_extract).  A plan becomes degree maps once (cached per
# plan on the device): maps[kind][d] = source element of degree d (encode) or destination of product
# coefficient d (decode), -1 where nothing goes.  A whole job -- or a batch of jobs -- is then one
# descriptor: polynomial p reads src[base[p] + maps[kind[p]][d]].

@dataclasses.dataclass
class Gather:
    """Encode descriptor of n polynomials: flat int64 source values plus per-polynomial (kind, base)."""

    src: torch.Tensor       # flat int64 (signed values, reduced mod t by the kernel)
    maps: torch.Tensor      # [K, N] int32
    kind: torch.Tensor      # [P] int32
    base: torch.Tensor      # [P] int64

    @property
    def n_polys(self) -> int:
        return int(self.kind.shape[0])


@dataclasses.dataclass
class Scatter:
    """Decode descriptor: product coefficient d of slot s lands at base[s] + maps[kind[s]][d]."""

    maps: torch.Tensor
    kind: torch.Tensor
    base: torch.Tensor
    shape: tuple            # output tensor shape (numel = prod(shape))

    @property
    def numel(self) -> int:
        return int(np.prod(self.shape)) if self.shape else 1


def _dev_i32(a) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()


def _dev_i64(a) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).cuda()


def input_maps(plan: PackingPlan) -> np.ndarray:
    """[tiles, N]: source offset (within one H x W channel) of every packed input degree."""
    t_ids, degs, srcs = input_index_map(plan)
    maps = np.full((plan.num_tiles, plan.n), -1, dtype=np.int32)
    maps[t_ids, degs] = srcs
    return maps


def kernel_maps(plan: PackingPlan) -> np.ndarray:
    maps = np.full((1, plan.n), -1, dtype=np.int32)
    maps[0, kernel_degrees(plan)] = np.arange(plan.shape.kernel ** 2)
    return maps


def output_maps(plan: PackingPlan) -> np.ndarray:
    """[tiles, N]: destination (within one cropped output map) of every extracted degree."""
    t_ids, degs, dsts = output_index_map(plan)
    maps = np.full((plan.num_tiles, plan.n), -1, dtype=np.int32)
    maps[t_ids, degs] = dsts
    return maps


@functools.lru_cache(maxsize=256)
def _plan_maps_device(plan: PackingPlan, n: int) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """(input maps, kernel maps, output maps) of a plan on the device, padded to ring degree n."""
    def pad(m):
        if m.shape[1] == n:
            return m
        out = np.full((m.shape[0], n), -1, dtype=np.int32)
        out[:, :m.shape[1]] = m
        return out
    return _dev_i32(pad(input_maps(plan))), _dev_i32(pad(kernel_maps(plan))), _dev_i32(pad(output_maps(plan)))


@functools.lru_cache(maxsize=256)
def _fc_maps_device(n: int, in_dim: int, out_dim: int):
    """FC / outer-product degree maps (packing.py:545-605) for ring degree n: (input x at degree i,
    matrix group rows reversed at stride in_dim, fc output degrees r*in+in-1, outer left g[r] at
    degree r*in, outer output degrees r*in + j).  The grouped maps have two rows: row 0 for a full
    group of cap rows, row 1 for the last group, which holds only out_dim - (groups-1)*cap rows
    (extract_fc_output's `take`, packing.py:581-583) -- so a batch of jobs never reads or writes
    across an image boundary."""
    cap = fc_row_capacity(n, in_dim)
    groups = math.ceil(out_dim / cap)
    take = out_dim - (groups - 1) * cap
    d = np.arange(n)
    x_map = np.where(d < in_dim, d, -1)[None]
    r, k = d // in_dim, d % in_dim
    rows = []
    for lim in (cap, take):
        used = (d < cap * in_dim) & (r < lim)
        rows.append((np.where(used, r * in_dim + (in_dim - 1 - k), -1),
                     np.where(used & (k == in_dim - 1), r, -1),
                     np.where(used & (k == 0), r, -1),
                     np.where(used, d, -1)))
    w_map, fc_out, g_map, outer_out = (np.stack([rows[0][i], rows[1][i]]) for i in range(4))
    return tuple(_dev_i32(m) for m in (x_map, w_map, fc_out, g_map, outer_out))


def _group_kinds(groups: int, batch: int) -> np.ndarray:
    """Map row per group polynomial: 0 for full groups, 1 for the last group of each job."""
    k = np.zeros((batch, groups), dtype=np.int32)
    k[:, -1] = 1
    return k.ravel()


def _check_ctx(ctx):
    if not getattr(ctx, "t", 0):
        raise PackingError("packing needs a context with the plain ring")


def gather(ctx, side: Gather, r: torch.Tensor | None = None, want_plain: bool = True):
    """Run ctb_pack_gather: -> plain [P, N] int64 (and masked = plain - r mod t when r is given)."""
    from . import _lib
    from .device import _ptr, _stream
    _check_ctx(ctx)
    P, n = side.n_polys, ctx.n
    plain = torch.empty((P, n), dtype=torch.int64, device="cuda") if want_plain or r is None else None
    masked = None
    if r is not None:
        if tuple(r.shape) != (P, n):
            raise PackingError(f"mask shape {tuple(r.shape)} != {(P, n)}")
        masked = torch.empty((P, n), dtype=torch.int64, device="cuda")
    src = side.src.contiguous()
    _lib.check(ctx._lib.ctb_pack_gather(ctx._h, _ptr(src) if src.numel() else None, src.numel(), _ptr(side.maps),
                                        side.maps.shape[0], _ptr(side.kind), _ptr(side.base),
                                        _ptr(r.contiguous()) if r is not None else None,
                                        _ptr(plain) if plain is not None else None,
                                        _ptr(masked) if masked is not None else None, P, _stream()), "ctb_pack_gather")
    return plain if r is None else (plain, masked)


def scatter(ctx, values: torch.Tensor, out: Scatter, sub: torch.Tensor | None = None,
            centered: bool = False) -> torch.Tensor:
    """Run ctb_plain_scatter: [S, N] plain values (minus sub) -> tensor of out.shape (int64)."""
    from . import _lib
    from .device import _ptr, _stream
    _check_ctx(ctx)
    S = int(out.kind.shape[0])
    if values.shape[0] != S:
        raise PackingError(f"expected {S} products, got {values.shape[0]}")
    res = torch.zeros(out.shape, dtype=torch.int64, device="cuda")
    v = values.contiguous()
    _lib.check(ctx._lib.ctb_plain_scatter(ctx._h, _ptr(v), _ptr(sub.contiguous()) if sub is not None else None,
                                          _ptr(out.maps), out.maps.shape[0], _ptr(out.kind), _ptr(out.base),
                                          out.numel, int(centered), _ptr(res), S, _stream()), "ctb_plain_scatter")
    return res


# ------------------------------------------------------------------------- descriptors of the job families
#
# (kind, base) arrays depend only on the job's dimensions, so they are built once per dimension
# tuple and kept on the device: rebuilding a job of a known shape launches nothing and copies
# nothing until its gather / scatter kernel runs.

_DESC: dict = {}


def _kind_base(key: tuple, build) -> tuple[torch.Tensor, torch.Tensor]:
    hit = _DESC.get(key)
    if hit is None:
        kind, base = build()
        hit = (_dev_i32(kind), _dev_i64(base))
        if len(_DESC) > 4096:
            _DESC.clear()
        _DESC[key] = hit
    return hit


def _flat(x: torch.Tensor) -> torch.Tensor:
    return x.reshape(-1).to(torch.int64)


def conv_input_side(x: torch.Tensor, plan: PackingPlan, n: int) -> Gather:
    """x [..., H, W] -> polys ordered (leading index, tile) (packing.py:407-426 per channel)."""
    _check_plan_n(plan, n)
    sh = plan.shape
    if tuple(x.shape[-2:]) != (sh.height, sh.width):
        raise PackingError(f"input shape {tuple(x.shape[-2:])} != {(sh.height, sh.width)}")
    lead = int(np.prod(x.shape[:-2])) if x.dim() > 2 else 1
    T = plan.num_tiles
    imaps, _, _ = _plan_maps_device(plan, n)
    kind, base = _kind_base(("cin", T, lead, sh.height * sh.width), lambda: (
        np.tile(np.arange(T), lead), np.repeat(np.arange(lead, dtype=np.int64) * (sh.height * sh.width), T)))
    return Gather(_flat(x), imaps, kind, base)


def conv_kernel_side(w: torch.Tensor, plan: PackingPlan, n: int, repeat: int = 1) -> Gather:
    """w [..., h, h] -> one poly per leading index (packing.py:429-445), the whole sequence
    repeated `repeat` times (the same kernels packed for every image of a batch)."""
    _check_plan_n(plan, n)
    h = plan.shape.kernel
    if tuple(w.shape[-2:]) != (h, h):
        raise PackingError(f"kernel shape {tuple(w.shape[-2:])} != {(h, h)}")
    lead = int(np.prod(w.shape[:-2])) if w.dim() > 2 else 1
    _, kmaps, _ = _plan_maps_device(plan, n)
    kind, base = _kind_base(("ker", lead, repeat, h), lambda: (
        np.zeros(lead * repeat), np.tile(np.arange(lead, dtype=np.int64) * h * h, repeat)))
    return Gather(_flat(w), kmaps, kind, base)


@functools.lru_cache(maxsize=256)
def _strided_output_maps(plan: PackingPlan, n: int, stride: int) -> torch.Tensor:
    """Output maps of the stride-s convolution lowered as stride 1 + subsampling (
    not in the reference): only outputs (u, v) with u, v = 0 mod s are kept, at (u/s, v/s)."""
    sh = plan.shape
    ow = sh.out_width
    ow_s = -(-ow // stride)
    t_ids, degs, dsts = output_index_map(plan)
    u, v = dsts // ow, dsts % ow
    keep = (u % stride == 0) & (v % stride == 0)
    maps = np.full((plan.num_tiles, n), -1, dtype=np.int32)
    maps[t_ids[keep], degs[keep]] = (u[keep] // stride) * ow_s + v[keep] // stride
    return _dev_i32(maps)


def conv_output_side(plan: PackingPlan, n: int, maps_count: int, lead: tuple, stride: int = 1) -> Scatter:
    """Slots ordered (map index, tile) -> tensor lead + (out_h, out_w) (stride > 1: the subsampled
    output of the stride-1 job, (ceil(out_h/s), ceil(out_w/s)))."""
    sh = plan.shape
    T = plan.num_tiles
    oh, ow = -(-sh.out_height // stride), -(-sh.out_width // stride)
    omaps = _plan_maps_device(plan, n)[2] if stride == 1 else _strided_output_maps(plan, n, stride)
    kind, base = _kind_base(("out", T, maps_count, oh * ow), lambda: (
        np.tile(np.arange(T), maps_count), np.repeat(np.arange(maps_count, dtype=np.int64) * (oh * ow), T)))
    return Scatter(omaps, kind, base, tuple(lead) + (oh, ow))


def _check_plan_n(plan: PackingPlan, n: int):
    if plan.scheme != SCHEME_CORRELATED:
        raise PackingError(f"plan is for scheme {plan.scheme!r}, not {SCHEME_CORRELATED!r}")
    if plan.n > n:
        raise PackingError("plan degree budget exceeds the ring degree")
    if plan.degree_bound >= n:
        raise PackingOverflowError(f"plan needs degree {plan.degree_bound}, ring has {n}")


# ------------------------------------------------------------------------- batched device packing

def pack_input_batch(x: torch.Tensor, plan: PackingPlan, params: RingParams) -> torch.Tensor:
    """x [..., H, W] signed ints -> [..., tiles, N] plain values in [0, t)."""
    from .ring import context_of
    _check_plan(plan, params)
    side = conv_input_side(x, plan, params.n)
    out = gather(context_of(params), side)
    return out.view(*x.shape[:-2], plan.num_tiles, params.n)


def pack_kernel_batch(w: torch.Tensor, plan: PackingPlan, params: RingParams) -> torch.Tensor:
    """w [..., h, h] signed ints -> [..., N] plain values."""
    from .ring import context_of
    _check_plan(plan, params)
    side = conv_kernel_side(w, plan, params.n)
    return gather(context_of(params), side).view(*w.shape[:-2], params.n)


def extract_batch(products: torch.Tensor, plan: PackingPlan, params: RingParams,
                  centered: bool = False) -> torch.Tensor:
    """[..., tiles, N] product coefficients (mod t) -> [..., out_h, out_w] (residues, or centred)."""
    from .ring import context_of
    if plan.degree_bound >= products.shape[-1]:
        raise PackingOverflowError(f"plan uses degree {plan.degree_bound} >= ring degree {products.shape[-1]}: wrapped")
    if products.shape[-2] != plan.num_tiles:
        raise PackingError(f"expected {plan.num_tiles} products, got {products.shape[-2]}")
    n = products.shape[-1]
    lead = tuple(products.shape[:-2])
    maps_count = int(np.prod(lead)) if lead else 1
    out = conv_output_side(plan, n, maps_count, lead)
    return scatter(context_of(params), products.reshape(-1, n), out, centered=centered)


# ------------------------------------------------------------------------- reference-shaped API

def pack_input_correlated(x, shape: ConvShape, params: RingParams, plan: PackingPlan | None = None):
    plan = plan or plan_correlated(shape, params.n)
    xt = torch.as_tensor(np.asarray(x, dtype=np.int64), device="cuda")
    polys = pack_input_batch(xt, plan, params)
    return [RingElem(params, polys[t].contiguous()) for t in range(plan.num_tiles)], plan


def pack_kernel_correlated(w, shape: ConvShape, params: RingParams, plan: PackingPlan | None = None):
    plan = plan or plan_correlated(shape, params.n)
    wt = torch.as_tensor(np.asarray(w, dtype=np.int64), device="cuda")
    return RingElem(params, pack_kernel_batch(wt, plan, params).contiguous()), plan


def extract_output(products, plan: PackingPlan) -> np.ndarray:
    if len(products) != plan.num_tiles:
        raise PackingError(f"expected {plan.num_tiles} products, got {len(products)}")
    stacked = torch.stack([p.data for p in products])
    return extract_batch(stacked, plan, products[0].params).cpu().numpy().astype(np.uint64)


def to_signed_matrix(mat, modulus: int) -> np.ndarray:
    mat = np.asarray(mat)
    half = modulus // 2
    if mat.dtype != object and modulus < (1 << 62):
        v = mat.astype(np.int64) % np.int64(modulus)
        return np.where(v > half, v - modulus, v)
    out = mat.astype(object) % modulus
    return np.where(out > half, out - modulus, out)


def to_signed_tensor(t: torch.Tensor, modulus: int) -> torch.Tensor:
    v = torch.remainder(t, modulus)
    return torch.where(v > modulus // 2, v - modulus, v)


# ------------------------------------------------------------------------- fully connected (packing.py:541-605)

def fc_row_capacity(n: int, in_dim: int) -> int:
    return max(1, n // in_dim)


def fc_input_side(x: torch.Tensor, n: int) -> Gather:
    """x [..., d] (d <= N) -> one poly per leading index, x[i] at degree i (packing.py:545-550)."""
    d = x.shape[-1]
    if d > n:
        raise PackingError(f"fc input dimension {d} exceeds ring degree")
    lead = int(np.prod(x.shape[:-1])) if x.dim() > 1 else 1
    kind, base = _kind_base(("fcx", lead, d), lambda: (np.zeros(lead), np.arange(lead, dtype=np.int64) * d))
    return Gather(_flat(x), _fc_maps_device(n, d, 1)[0], kind, base)


def fc_matrix_side(w: torch.Tensor, n: int, repeat: int = 1) -> Gather:
    """w [out, in] -> ceil(out / cap) polys, rows reversed at stride in_dim (packing.py:553-574);
    the groups repeated `repeat` times (one copy per image of a batch)."""
    out_dim, in_dim = w.shape[-2:]
    if in_dim > n:
        raise PackingError(f"fc input dimension {in_dim} exceeds ring degree")
    cap = fc_row_capacity(n, in_dim)
    groups = math.ceil(out_dim / cap)
    kind, base = _kind_base(("fcw", groups, repeat, cap * in_dim), lambda: (
        _group_kinds(groups, repeat), np.tile(np.arange(groups, dtype=np.int64) * cap * in_dim, repeat)))
    return Gather(_flat(w), _fc_maps_device(n, in_dim, out_dim)[1], kind, base)


def fc_output_side(n: int, out_dim: int, in_dim: int, batch: int = 1, lead: tuple = ()) -> Scatter:
    """Row r of group g lands at b * out_dim + g * cap + r (extract_fc_output, packing.py:577-586)."""
    cap = fc_row_capacity(n, in_dim)
    groups = math.ceil(out_dim / cap)
    kind, base = _kind_base(("fco", groups, batch, cap, out_dim), lambda: (
        _group_kinds(groups, batch),
        (np.arange(batch, dtype=np.int64)[:, None] * out_dim + np.arange(groups) * cap).ravel()))
    return Scatter(_fc_maps_device(n, in_dim, out_dim)[2], kind, base, tuple(lead) + (out_dim,))


def outer_left_side(g: torch.Tensor, in_dim: int, n: int) -> Gather:
    """g [..., m] -> per leading index ceil(m / cap) polys with g[r] at degree r * in_dim
    (packing.py:589-599)."""
    cap = fc_row_capacity(n, in_dim)
    m = g.shape[-1]
    lead = int(np.prod(g.shape[:-1])) if g.dim() > 1 else 1
    groups = math.ceil(m / cap)
    kind, base = _kind_base(("ogl", lead, groups, m, cap), lambda: (
        _group_kinds(groups, lead), (np.arange(lead, dtype=np.int64)[:, None] * m + np.arange(groups) * cap).ravel()))
    return Gather(_flat(g), _fc_maps_device(n, in_dim, m)[3], kind, base)


def outer_output_side(n: int, out_dim: int, in_dim: int, batch: int = 1, lead: tuple = ()) -> Scatter:
    """Group j of image b lands at (b * out_dim + j * cap) * in_dim + d (extract_outer, :602-605)."""
    cap = fc_row_capacity(n, in_dim)
    groups = math.ceil(out_dim / cap)
    kind, base = _kind_base(("ogo", batch, groups, out_dim, cap, in_dim), lambda: (
        _group_kinds(groups, batch),
        ((np.arange(batch, dtype=np.int64)[:, None] * out_dim + np.arange(groups) * cap) * in_dim).ravel()))
    return Scatter(_fc_maps_device(n, in_dim, out_dim)[4], kind, base, tuple(lead) + (out_dim, in_dim))


def pack_fc_input_batch(x: torch.Tensor, params: RingParams) -> torch.Tensor:
    """x [..., d] (d <= N) -> [..., N]: x[i] at degree i."""
    from .ring import context_of
    side = fc_input_side(x, params.n)
    return gather(context_of(params), side).view(*x.shape[:-1], params.n)


def pack_fc_matrix_batch(w: torch.Tensor, params: RingParams) -> torch.Tensor:
    """w [out, in] -> [groups, N]: row r of a group reversed at degrees r*in .. r*in+in-1."""
    from .ring import context_of
    return gather(context_of(params), fc_matrix_side(w, params.n))
