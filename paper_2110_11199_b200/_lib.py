"""ctypes binding of libadpsgd_b200.so (the C ABI declared in include/adpsgd_b200.h).

There is no fallback: if the CUDA library is missing this module raises on load.
"""
from __future__ import annotations

import ctypes as C
import os
import re

from .errors import raise_for

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG_DIR)
# ADPSGD_LIB_PATH: an alternative build of the same library (A/B timing experiments, tools/ab.sh)
LIB_PATH = os.environ.get("ADPSGD_LIB_PATH") or os.path.join(PKG_DIR, "libadpsgd_b200.so")
HEADER = os.path.join(ROOT, "include", "adpsgd_b200.h")

u64, i64, i32 = C.c_uint64, C.c_int64, C.c_int32
P = C.POINTER


class ModelDesc(C.Structure):
    _fields_ = [(n, i32) for n in
                ("layers", "hidden", "bidirectional", "input_dim", "proj", "classes", "unroll")]


class Config(C.Structure):
    _fields_ = [("model", ModelDesc), ("precision", i32), ("strategy", i32), ("learners", i32),
                ("first_learner", i32), ("local_learners", i32), ("batch", i32), ("device", i32),
                ("generic_mix", i32), ("staleness_cap", i32), ("seed", u64)]


class Perf(C.Structure):
    _fields_ = [("last_step_ms", C.c_double), ("last_mix_ms", C.c_double), ("gossip_bytes", C.c_double),
                ("steps", i64), ("kernel_launches", i64), ("comm_start_ms", C.c_double),
                ("comm_end_ms", C.c_double), ("compute_end_ms", C.c_double)]


class AsyncInfo(C.Structure):
    _fields_ = [("version", i64), ("left_version", i64), ("right_version", i64), ("left", i32), ("right", i32),
                ("retries", i32), ("reserved", i32), ("wait_ms", C.c_double), ("step_ms", C.c_double)]


class AsyncRecord(C.Structure):  # adpsgd_async_record
    _fields_ = [("heldout_idx", P(i32)), ("n_heldout", i32), ("train_idx", P(i32)), ("n_train", i32),
                ("initial_heldout", C.c_double), ("consensus", P(C.c_double)), ("cap_iters", i64),
                ("heldout", P(C.c_double)), ("train", P(C.c_double)), ("cap_epochs", i32), ("n_iters", i64),
                ("n_epochs", i32), ("diverged_epoch", i32)]


_SIGS = {
    "adpsgd_param_count": (i64, [P(ModelDesc)]),
    "adpsgd_permutation_for_iteration": (C.c_int, [u64, i32, i64, P(i32)]),
    "adpsgd_pairing": (C.c_int, [i32, u64, i32, i64, P(i32), P(i32)]),
    "adpsgd_lr_at": (C.c_double, [C.c_double, C.c_double, i32, C.c_double, i32, i32]),
    "adpsgd_last_error": (C.c_char_p, []),
    "adpsgd_build_info": (C.c_char_p, []),
    "adpsgd_ctx_create": (C.c_int, [P(Config), P(C.c_void_p)]),
    "adpsgd_ctx_destroy": (C.c_int, [C.c_void_p]),
    "adpsgd_set_dataset": (C.c_int, [C.c_void_p, P(C.c_float), P(i32), i32, i32]),
    "adpsgd_synth_dataset": (C.c_int, [C.c_void_p, i32, i32, u64]),
    "adpsgd_get_dataset": (C.c_int, [C.c_void_p, P(C.c_float), P(i32)]),
    "adpsgd_set_weights": (C.c_int, [C.c_void_p, i32, P(C.c_double), i64]),
    "adpsgd_get_weights": (C.c_int, [C.c_void_p, i32, P(C.c_double), i64]),
    "adpsgd_step": (C.c_int, [C.c_void_p, C.c_double, P(i32), P(C.c_float)]),
    "adpsgd_step_host_batch": (C.c_int, [C.c_void_p, C.c_double, P(C.c_float), P(i32), P(C.c_float)]),
    "adpsgd_prefetch_host_batch": (C.c_int, [C.c_void_p, P(C.c_float), P(i32)]),
    "adpsgd_debug_buffer": (C.c_int, [C.c_void_p, i32, C.c_void_p, C.c_size_t]),
    "adpsgd_debug_buffer_range": (C.c_int, [C.c_void_p, i32, P(u64), P(u64)]),
    "adpsgd_step_injected": (C.c_int, [C.c_void_p, C.c_double, P(i32), P(C.c_double)]),
    "adpsgd_gradient": (C.c_int, [C.c_void_p, P(C.c_double), P(i32), i32, P(C.c_double), P(C.c_double)]),
    "adpsgd_set_straggler": (C.c_int, [C.c_void_p, i32, C.c_double]),
    "adpsgd_get_stats": (C.c_int, [C.c_void_p, P(Perf)]),
    "adpsgd_iteration": (i64, [C.c_void_p]),
    "adpsgd_set_iteration": (C.c_int, [C.c_void_p, i64]),
    "adpsgd_consensus_distance": (C.c_int, [C.c_void_p, P(C.c_double)]),
    "adpsgd_eval_loss": (C.c_int, [C.c_void_p, P(C.c_double), P(i32), i32, P(C.c_double)]),
    "adpsgd_averaged_model": (C.c_int, [C.c_void_p, P(C.c_double), i64]),
    "adpsgd_consensus_gram": (C.c_int, [C.c_void_p, i64, i64, P(C.c_double)]),
    "adpsgd_consensus_from_gram": (C.c_int, [P(C.c_double), i32, P(C.c_double)]),
    "adpsgd_averaged_model_all": (C.c_int, [C.c_void_p, P(C.c_double), i64]),
    "adpsgd_async_run": (C.c_int, [C.c_void_p, i32, P(C.c_double), i64, i32, P(C.c_double), i32, P(i32),
                                   P(C.c_double), P(i64)]),
    "adpsgd_async_run_record": (C.c_int, [C.c_void_p, i32, P(C.c_double), i64, i32, P(C.c_double), i32, P(i32),
                                          P(C.c_double), P(AsyncRecord), P(i64)]),
    "adpsgd_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "adpsgd_comm_init": (C.c_int, [C.c_void_p, i32, i32, C.c_void_p]),
    "adpsgd_ipc_handle_size": (i64, [C.c_void_p]),
    "adpsgd_export_ipc": (C.c_int, [C.c_void_p, C.c_void_p, i64]),
    "adpsgd_import_ipc": (C.c_int, [C.c_void_p, i32, i32, i32, C.c_void_p, i64]),
    "adpsgd_set_gossip_mode": (C.c_int, [C.c_void_p, i32]),
    "adpsgd_barrier": (C.c_int, [C.c_void_p]),
    "adpsgd_group_link": (C.c_int, [P(C.c_void_p), i32]),
    "adpsgd_group_step": (C.c_int, [P(C.c_void_p), i32, C.c_double, P(C.c_float)]),
    "adpsgd_async_init": (C.c_int, [C.c_void_p, i32, i32, C.c_double]),
    "adpsgd_async_step": (C.c_int, [C.c_void_p, C.c_double, P(C.c_float), P(AsyncInfo)]),
    "adpsgd_set_step_delay": (C.c_int, [C.c_void_p, i32, C.c_double, i32]),
    "adpsgd_gossip_probe": (C.c_int, [C.c_void_p, i32, i32, i32, P(C.c_double)]),
    "adpsgd_profile_enable": (C.c_int, [i32]),
    "adpsgd_profile_read": (C.c_int, [P(C.c_double), P(C.c_double), P(C.c_double), P(i64), i32]),
    "adpsgd_kernel_variants": (C.c_int, [C.c_char_p, C.c_size_t, i32]),
    "adpsgd_debug_trace": (C.c_int, [i32, C.c_void_p, i32]),
    "adpsgd_gemm": (C.c_int, [i32, i32, i32, i32, C.c_void_p, i64, i32, C.c_void_p, i64, i32, C.c_void_p, i64,
                              i32, C.c_float, i32, C.c_void_p, C.c_void_p]),
    "adpsgd_mix_update": (C.c_int, [i64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_float, C.c_void_p,
                                    C.c_void_p, C.c_void_p]),
}

PROF_CATS = ["gemm_rec_fwd", "gemm_rec_bwd", "gemm_wgrad", "gemm_dgrad_x", "gemm_out", "gemm_simt", "lstm_cell",
             "softmax_ce", "reduce", "gather", "mix_update", "other"]
GEMM_TC_CATS = PROF_CATS[:5]

_LIB = None


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    with open(HEADER) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z0-9_]+\s*\**\s*(adpsgd_[a-z0-9_]+)\s*\(", text, flags=re.M)))


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def last_error() -> str:
    msg = lib().adpsgd_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    if rc != 0:
        raise_for(rc, last_error())


def profile_enable(on: bool) -> None:
    check(lib().adpsgd_profile_enable(int(on)))


def profile_read() -> dict:
    n = len(PROF_CATS)
    ms, fl, by = (C.c_double * n)(), (C.c_double * n)(), (C.c_double * n)()
    la = (C.c_int64 * n)()
    check(lib().adpsgd_profile_read(ms, fl, by, la, n))
    return {c: {"ms": ms[i], "flops": fl[i], "bytes": by[i], "launches": la[i]} for i, c in enumerate(PROF_CATS)}


def kernel_variants(reset: bool = True) -> dict:
    """Kernel variants (tcgen05 template instantiations) selected since the last reset, with the
    number of times each was chosen (eager launches and graph captures; replays are not counted)."""
    buf = C.create_string_buffer(1 << 16)
    check(lib().adpsgd_kernel_variants(buf, len(buf), int(reset)))
    out = {}
    for item in buf.value.decode().split(";"):
        if item:
            name, _, n = item.rpartition("=")
            out[name] = int(n)
    return out
