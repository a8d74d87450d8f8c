"""Correlated tensor <-> polynomial packing (mirror of privtrain.packing, correlated scheme).

Input entry (i, j) of a window starting at (r0, c0) goes to degree
(i - r0) * O + (j - c0) with row stride O = max(window) + h - 1, kernel entry
(i, j) to degree (h-1-i) * O + (h-1-j); every product coefficient at degree
u * O + v is then an output of the full-padding convolution
(packing.py:11-16, 407-509 in the reference).  Window selection is the
reference's exhaustive minimum-tile-count search with the same tie-break
(packing.py:225-260), so plans -- and therefore sites and ciphertexts -- are
identical.

The device path packs and extracts whole batches with one index scatter /
gather each (`pack_input_batch`, `extract_batch`); the per-polynomial
functions keep the reference's signatures and return device RingElems.
The row-major "baseline" scheme and the analytic count report are
reference-side experiments outside the hot path.
"""
from __future__ import annotations

import dataclasses
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


def _to_mod(vals: torch.Tensor, modulus: int) -> torch.Tensor:
    return torch.remainder(vals.to(torch.int64), modulus)


# ------------------------------------------------------------------------- batched device packing

def pack_input_batch(x: torch.Tensor, plan: PackingPlan, params: RingParams) -> torch.Tensor:
    """x [..., H, W] signed ints -> [..., tiles, N] plain values in [0, t)."""
    _check_plan(plan, params)
    sh = plan.shape
    if tuple(x.shape[-2:]) != (sh.height, sh.width):
        raise PackingError(f"input shape {tuple(x.shape[-2:])} != {(sh.height, sh.width)}")
    lead = x.shape[:-2]
    t_ids, degs, srcs = (torch.as_tensor(a, device=x.device) for a in input_index_map(plan))
    flat = _to_mod(x.reshape(-1, sh.height * sh.width), params.modulus)
    out = torch.zeros((flat.shape[0], plan.num_tiles * params.n), dtype=torch.int64, device=x.device)
    out[:, t_ids * params.n + degs] = flat[:, srcs]
    return out.view(*lead, plan.num_tiles, params.n)


def pack_kernel_batch(w: torch.Tensor, plan: PackingPlan, params: RingParams) -> torch.Tensor:
    """w [..., h, h] signed ints -> [..., N] plain values."""
    _check_plan(plan, params)
    h = plan.shape.kernel
    if tuple(w.shape[-2:]) != (h, h):
        raise PackingError(f"kernel shape {tuple(w.shape[-2:])} != {(h, h)}")
    lead = w.shape[:-2]
    flat = _to_mod(w.reshape(-1, h * h), params.modulus)
    out = torch.zeros((flat.shape[0], params.n), dtype=torch.int64, device=w.device)
    out[:, torch.as_tensor(kernel_degrees(plan), device=w.device)] = flat
    return out.view(*lead, params.n)


def extract_batch(products: torch.Tensor, plan: PackingPlan) -> torch.Tensor:
    """[..., tiles, N] product coefficients -> [..., out_h, out_w] (mod-t residues)."""
    if plan.degree_bound >= products.shape[-1]:
        raise PackingOverflowError(f"plan uses degree {plan.degree_bound} >= ring degree {products.shape[-1]}: wrapped")
    if products.shape[-2] != plan.num_tiles:
        raise PackingError(f"expected {plan.num_tiles} products, got {products.shape[-2]}")
    sh = plan.shape
    n = products.shape[-1]
    lead = products.shape[:-2]
    t_ids, degs, dsts = (torch.as_tensor(a, device=products.device) for a in output_index_map(plan))
    src = products.reshape(-1, plan.num_tiles * n)
    out = torch.zeros((src.shape[0], sh.out_height * sh.out_width), dtype=products.dtype, device=products.device)
    out[:, dsts] = src[:, t_ids * n + degs]
    return out.view(*lead, sh.out_height, sh.out_width)


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
    stacked = torch.stack([p.data for p in products])
    return extract_batch(stacked, plan).cpu().numpy().astype(np.uint64)


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


def pack_fc_input_batch(x: torch.Tensor, params: RingParams) -> torch.Tensor:
    """x [..., d] (d <= N) -> [..., N]: x[i] at degree i."""
    d = x.shape[-1]
    if d > params.n:
        raise PackingError(f"fc input dimension {d} exceeds ring degree")
    out = torch.zeros((*x.shape[:-1], params.n), dtype=torch.int64, device=x.device)
    out[..., :d] = _to_mod(x, params.modulus)
    return out


def pack_fc_matrix_batch(w: torch.Tensor, params: RingParams) -> torch.Tensor:
    """w [out, in] -> [groups, N]: row r of a group reversed at degrees r*in .. r*in+in-1."""
    out_dim, in_dim = w.shape[-2:]
    if in_dim > params.n:
        raise PackingError(f"fc input dimension {in_dim} exceeds ring degree")
    cap = fc_row_capacity(params.n, in_dim)
    groups = math.ceil(out_dim / cap)
    rows = torch.zeros((groups * cap, in_dim), dtype=torch.int64, device=w.device)
    rows[:out_dim] = _to_mod(w.flip(-1), params.modulus)
    out = torch.zeros((groups, params.n), dtype=torch.int64, device=w.device)
    out[:, :cap * in_dim] = rows.view(groups, cap * in_dim)
    return out


def extract_fc_batch(products: torch.Tensor, out_dim: int, in_dim: int) -> torch.Tensor:
    n = products.shape[-1]
    cap = fc_row_capacity(n, in_dim)
    degs = torch.arange(cap, device=products.device) * in_dim + (in_dim - 1)
    vals = products[..., degs].reshape(*products.shape[:-2], -1)
    return vals[..., :out_dim]


def pack_outer_left_batch(g: torch.Tensor, in_dim: int, params: RingParams) -> torch.Tensor:
    """g [m] -> [groups, N] with g[r] at degree r * in_dim (per group)."""
    cap = fc_row_capacity(params.n, in_dim)
    m = g.shape[-1]
    groups = math.ceil(m / cap)
    out = torch.zeros((groups, params.n), dtype=torch.int64, device=g.device)
    padded = torch.zeros(groups * cap, dtype=torch.int64, device=g.device)
    padded[:m] = _to_mod(g, params.modulus)
    out[:, torch.arange(cap, device=g.device) * in_dim] = padded.view(groups, cap)
    return out


def extract_outer_batch(products: torch.Tensor, out_dim: int, in_dim: int) -> torch.Tensor:
    n = products.shape[-1]
    cap = fc_row_capacity(n, in_dim)
    vals = products[..., :cap * in_dim].reshape(*products.shape[:-2], -1, in_dim)
    return vals[..., :out_dim, :]
