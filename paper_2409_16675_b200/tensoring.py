"""CCMul on device: exact tensoring and relinearisation (he.py:384-432).

Thin batching wrappers over ctb_ccmul_raw / ctb_relinearize; the batch is cut
into chunks so the uint32 workspace (7 K N words per ciphertext pair, K = 17
auxiliary primes at N = 4096) stays bounded.
"""
from __future__ import annotations

import torch

from . import _lib
from .device import RnsContext, _ptr, _stream

WORKSPACE_BYTES = 512 << 20


def _chunk(ctx: RnsContext, per_item_words: int) -> int:
    return max(1, WORKSPACE_BYTES // (4 * max(1, per_item_words)))


def tensor_round(ctx: RnsContext, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """a, b [B, 2, L, N] -> [B, 3, L, N] = round((a (x) b) t / q) mod q."""
    B = a.shape[0]
    out = torch.empty((B, 3, ctx.L, ctx.n), dtype=a.dtype, device=a.device)
    per = int(ctx._lib.ctb_ccmul_workspace_words(ctx._h, 1))
    if per == 0:
        _lib.check(_lib.CTB_ERR_ARG, "ctb_ccmul_workspace_words")
    step = min(B, _chunk(ctx, per))
    ws = torch.empty(step * per, dtype=torch.int32, device=a.device)
    for s in range(0, B, step):
        e = min(B, s + step)
        _lib.check(ctx._lib.ctb_ccmul_raw(ctx._h, _ptr(a[s:e]), _ptr(b[s:e]), _ptr(out[s:e]), _ptr(ws), e - s,
                                          _stream()), "ctb_ccmul_raw")
    return out


def relinearize(ctx: RnsContext, ct3: torch.Tensor, keyprep: torch.Tensor) -> torch.Tensor:
    """ct3 [B, 3, L, N], keyprep [D, 2, L, N] (prepared) -> [B, 2, L, N]."""
    B = ct3.shape[0]
    D = ctx._lib.ctb_relin_digit_count(ctx._h)
    out = torch.empty((B, 2, ctx.L, ctx.n), dtype=ct3.dtype, device=ct3.device)
    step = min(B, _chunk(ctx, D * ctx.n))
    ws = torch.empty(step * D * ctx.n, dtype=torch.int32, device=ct3.device)
    for s in range(0, B, step):
        e = min(B, s + step)
        _lib.check(ctx._lib.ctb_relinearize(ctx._h, _ptr(ct3[s:e]), _ptr(keyprep), _ptr(ws), _ptr(out[s:e]), e - s,
                                            _stream()), "ctb_relinearize")
    return out
