"""ctypes binding of the C ABI in include/ctb200.h (libctb200.so, built in-tree).

There is deliberately no fallback: if the library is missing or no CUDA
device is visible, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libctb200.so"
# development A/B builds (tools/ab_variants.py) point CTB_LIB at an alternative in-tree build
if os.environ.get("CTB_LIB"):
    LIB_PATH = Path(os.environ["CTB_LIB"]).resolve()

CTB_OK, CTB_ERR_ARG, CTB_ERR_CUDA, CTB_ERR_UNSUPPORTED = 0, -1, -2, -3
BASE_Q, BASE_T, BASE_B = 0, 1, 2

_c_void_p = ctypes.c_void_p
_u64 = ctypes.c_uint64
_u32 = ctypes.c_uint32
_int = ctypes.c_int

# name -> (restype, argtypes); every symbol declared in include/ctb200.h
SIGNATURES: dict[str, tuple] = {
    "ctb_last_error": (ctypes.c_char_p, []),
    "ctb_version": (_int, []),
    "ctb_ctx_create": (_int, [ctypes.POINTER(_c_void_p), _u32, ctypes.POINTER(_u64), _u32,
                              ctypes.POINTER(_u64), _u32, _u32]),
    "ctb_ctx_destroy": (_int, [_c_void_p]),
    "ctb_ctx_word_bytes": (_int, [_c_void_p, _int]),
    "ctb_ctx_base_size": (_int, [_c_void_p, _int]),
    "ctb_ctx_base_primes": (_int, [_c_void_p, _int, ctypes.POINTER(_u64), _u32]),
    "ctb_ntt_forward": (_int, [_c_void_p, _int, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_ntt_inverse": (_int, [_c_void_p, _int, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_pointwise_mul": (_int, [_c_void_p, _int, _c_void_p, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_ring_mul": (_int, [_c_void_p, _int, _c_void_p, _u64, _c_void_p, _u64, _c_void_p, _u64, _c_void_p]),
    "ctb_prepare_operand": (_int, [_c_void_p, _int, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_mul_prepared": (_int, [_c_void_p, _int, _c_void_p, _c_void_p, _u64, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_mul_prepared_strided": (_int, [_c_void_p, _int, _c_void_p, _u64, _c_void_p, _u64, _c_void_p, _u64, _c_void_p, _u64,
                                         _c_void_p]),
    "ctb_cpmul": (_int, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_encrypt": (_int, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_encrypt_gather": (_int, [_c_void_p, _c_void_p, _u64, _c_void_p, _u32, _c_void_p, _c_void_p, _c_void_p, _c_void_p,
                                   _c_void_p, _u64, _c_void_p]),
    "ctb_sample_draws": (_int, [_c_void_p, _u64, _u64, ctypes.c_double, _int, _c_void_p, _u64, _c_void_p]),
    "ctb_draws_from_natural": (_int, [_c_void_p, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_pp_mul": (_int, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_rns_elementwise": (_int, [_c_void_p, _int, _int, _c_void_p, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_rns_scalar_mul": (_int, [_c_void_p, _int, _c_void_p, ctypes.POINTER(_u64), _c_void_p, _u64, _c_void_p]),
    "ctb_rns_from_small": (_int, [_c_void_p, _int, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_lift_plain": (_int, [_c_void_p, _c_void_p, ctypes.POINTER(_u64), _c_void_p, _u64, _c_void_p]),
    "ctb_plain_elementwise": (_int, [_c_void_p, _int, _c_void_p, _c_void_p, _u64, _c_void_p, _u64, _c_void_p]),
    "ctb_decrypt_round": (_int, [_c_void_p, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_decrypt_round_extract": (_int, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _u32, _c_void_p, _c_void_p, _u64,
                                          _int, _c_void_p, _u64, _c_void_p]),
    "ctb_pack_gather": (_int, [_c_void_p, _c_void_p, _u64, _c_void_p, _u32, _c_void_p, _c_void_p, _c_void_p, _c_void_p,
                               _c_void_p, _u64, _c_void_p]),
    "ctb_plain_scatter": (_int, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _u32, _c_void_p, _c_void_p, _u64, _int,
                                 _c_void_p, _u64, _c_void_p]),
    "ctb_bits_words": (_u64, [_u32, _u64]),
    "ctb_bits_pack": (_int, [_c_void_p, _int, _c_void_p, _u32, _c_void_p, _u64, _c_void_p]),
    "ctb_bits_unpack": (_int, [_c_void_p, _int, _c_void_p, _u32, _c_void_p, _u64, _c_void_p]),
    "ctb_ctx_pos_words": (_int, [_c_void_p]),
    "ctb_rns_to_pos": (_int, [_c_void_p, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_pos_to_rns": (_int, [_c_void_p, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_ccmul_workspace_words": (_u64, [_c_void_p, _u64]),
    "ctb_ccmul_raw": (_int, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_tensor_aux_size": (_int, [_c_void_p]),
    "ctb_tensor_lift": (_int, [_c_void_p, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_tensor_product": (_int, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_tensor_round": (_int, [_c_void_p, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_relin_digit_count": (_int, [_c_void_p]),
    "ctb_relinearize": (_int, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_lift_prepare": (_int, [_c_void_p, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_linear_online_workspace_bytes": (_u64, [_c_void_p, _u32, _u32, _u32, _u32]),
    "ctb_linear_online": (_int, [_c_void_p, _c_void_p, _u32, _c_void_p, _u32, _c_void_p, _c_void_p,
                                 ctypes.POINTER(_u32), _u32, _u32, _c_void_p, _int, _c_void_p, _c_void_p, _c_void_p,
                                 _c_void_p]),
    "ctb_eval_addend": (_int, [_c_void_p, _int, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_linear_addend": (_int, [_c_void_p, _int, _c_void_p, _c_void_p, _u64, _c_void_p]),
    "ctb_ccmul_sum_workspace_bytes": (_u64, [_c_void_p, _u32, _u32, _u32, _u32, _u32]),
    "ctb_ccmul_sum": (_int, [_c_void_p, _c_void_p, _u32, _c_void_p, _u32, _c_void_p, _u32, _u32, _c_void_p, _c_void_p,
                             _c_void_p, _u64, _c_void_p]),
    "ctb_slot_sum": (_int, [_c_void_p, _int, _c_void_p, _u32, _c_void_p, _c_void_p, _u32, _c_void_p, _c_void_p]),
    "ctb_probe_modmul": (_int, [_int, _u64, _c_void_p, ctypes.POINTER(_u64), _c_void_p]),
    "ctb_probe_modmul_mix": (_int, [_int, _u64, _c_void_p, ctypes.POINTER(_u64), _c_void_p]),
    "ctb_probe_modmul_mix_splice": (_int, [_int, _u64, _c_void_p, ctypes.POINTER(_u64), _c_void_p]),
    "ctb_probe_bfly_pass": (_int, [_c_void_p, _u64, _c_void_p, ctypes.POINTER(_u64), _c_void_p]),
    "ctb_probe_modmul_f64": (_int, [_u64, _c_void_p, ctypes.POINTER(_u64), _c_void_p]),
    "ctb_probe_bfly_f64": (_int, [_u64, _c_void_p, ctypes.POINTER(_u64), _c_void_p]),
    "ctb_check_f64q": (_int, [_c_void_p, _int, _u64, _u64, ctypes.POINTER(_u64), _c_void_p]),
}


class CtbError(RuntimeError):
    """A libctb200 call failed (argument, CUDA or unsupported-shape error)."""

    def __init__(self, code: int, what: str, msg: str):
        super().__init__(f"{what} failed ({code}): {msg}")
        self.code = code


_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def load() -> ctypes.CDLL:
    """Load libctb200.so once; raise loudly if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise CtbError(CTB_ERR_ARG, "load",
                               f"{LIB_PATH} is missing; build it with `python -m paper_2409_16675_b200.build`")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc != CTB_OK:
        msg = load().ctb_last_error()
        raise CtbError(rc, what, msg.decode() if msg else "")


def u64_array(values) -> ctypes.Array:
    vals = [int(v) for v in values]
    return (_u64 * max(1, len(vals)))(*vals)
