"""ctypes binding of ``libspdz_b200.so`` (C ABI declared in include/spdz_b200.h).

The product path has no CPU fallback: if the CUDA library is missing or no
device is visible, calls raise ``BackendUnavailable`` (backend.hpp:17).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

from . import errors

import os as _os

# SPDZ_B200_LIB: alternate build of the same library (reduction-variant experiments only)
LIB_PATH = Path(_os.environ.get("SPDZ_B200_LIB") or str(Path(__file__).resolve().parent / "libspdz_b200.so"))
MAX_PARTIES = 8
MAX_OPERANDS = 8  # SPDZ_MAX_OPERANDS

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p


class Share(C.Structure):  # spdz_share_t
    _fields_ = [("vals", vp), ("macs", vp), ("lanes", C.c_uint64)]


class Triple(C.Structure):  # spdz_triple_t
    _fields_ = [("a", Share), ("b", Share), ("c", Share)]


class MTriple(C.Structure):  # spdz_mtriple_t
    _fields_ = [("din", C.c_uint32), ("rows", C.c_uint32), ("a", Share), ("b", Share), ("c", Share)]


class Capability(C.Structure):  # spdz_capability_t
    _fields_ = [("name", C.c_char * 32), ("min_kernel_size", C.c_uint64), ("threads_per_block", C.c_uint32),
                ("executable", C.c_int32), ("sm_count", C.c_int32), ("device", C.c_int32)]


class BMTriple(C.Structure):  # spdz_bmtriple_t
    _fields_ = [("din", C.c_uint32), ("dout", C.c_uint32), ("batch", C.c_uint32), ("a", Share), ("b", Share),
                ("c", Share)]


class StoreInfo(C.Structure):  # spdz_store_info_t
    _fields_ = [("party", C.c_int32), ("n_parties", C.c_int32), ("alpha_share", C.c_uint32), ("loop_iters", C.c_uint64),
                ("scalar_triples", C.c_uint64), ("matrix_triples", C.c_uint64), ("input_masks", C.c_uint64)]


class MacSegment(C.Structure):  # spdz_mac_segment_t
    _fields_ = [("value", vp), ("mac_a", vp), ("mac_b", vp), ("len", C.c_uint64), ("j0", C.c_uint64),
                ("batch_id", C.c_uint64), ("lane0", C.c_uint64), ("batch_len", C.c_uint64)]


class Node(C.Structure):  # spdz_node_t
    _fields_ = [("kind", C.c_int32), ("is_private", C.c_int32), ("lanes", C.c_uint32), ("n_operands", C.c_uint32),
                ("operands", C.c_uint32 * MAX_OPERANDS), ("din", C.c_uint32), ("dout", C.c_uint32),
                ("const_val", C.c_uint32), ("next", C.c_uint32), ("loop_depth", C.c_uint32), ("n_succ", C.c_uint32),
                ("succ", C.c_uint32 * 2), ("phi_labels", C.c_uint32 * MAX_OPERANDS)]


class RunOptions(C.Structure):  # spdz_run_options_t
    _fields_ = [("slice", C.c_uint64), ("dealer_seed", C.c_uint64), ("fixed_coin", C.c_int32), ("coin", C.c_uint64),
                ("use_graph", C.c_int32), ("devices", C.c_int32 * MAX_PARTIES), ("profile_kernels", C.c_int32),
                ("stream_per_party", C.c_int32), ("shard_offset", C.c_uint64), ("shard_total", C.c_uint64),
                ("external_mac_verify", C.c_int32), ("single_party", C.c_int32), ("entry_label", C.c_uint32),
                ("loop_iters", C.c_uint64), ("network", C.c_int32), ("node_streams", C.c_int32),
                ("separate_party_kernels", C.c_int32), ("no_fusion", C.c_int32)]


class KernelStat(C.Structure):  # spdz_kernel_stat_t
    _fields_ = [("launches", C.c_uint64), ("ms", C.c_double), ("bytes", C.c_uint64)]


KSTAT_NAMES = ("mask", "combine", "sigma", "open")


class RunReport(C.Structure):  # spdz_run_report_t
    _fields_ = [("setup_ms", C.c_double), ("online_ms", C.c_double), ("online_device_ms", C.c_double),
                ("scalar_triples_consumed", C.c_uint64), ("matrix_triples_consumed", C.c_uint64),
                ("bytes_exchanged", C.c_uint64), ("output_digest", C.c_uint64), ("kernel_launches", C.c_uint64),
                ("sigmas", C.c_uint32 * MAX_PARTIES), ("coin", C.c_uint64), ("kstat", KernelStat * 4)]


_SIGS = {
    "spdz_last_error": (C.c_char_p, []),
    "spdz_version": (C.c_char_p, []),
    "spdz_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint32, C.POINTER(vp)]),
    "spdz_ctx_destroy": (C.c_int, [vp]),
    "spdz_ctx_set_stream": (C.c_int, [vp, vp]),
    "spdz_ctx_stream": (vp, [vp]),
    "spdz_ctx_use_own_stream": (C.c_int, [vp]),
    "spdz_ctx_party": (C.c_int, [vp]),
    "spdz_ctx_sync": (C.c_int, [vp]),
    "spdz_capability": (C.c_int, [vp, C.POINTER(Capability)]),
    "spdz_kernel_launches": (C.c_uint64, []),
    "spdz_diag_gemm_tc_flags": (C.c_int, [C.c_uint32]),
    "spdz_diag_gemm_tc_timeline": (C.c_int, [C.c_void_p]),
    "spdz_diag_imad_wide_rate": (C.c_int, [vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "spdz_diag_rep_check": (C.c_int, [vp, vp, C.c_uint64, vp]),
    "spdz_add_batch": (C.c_int, [vp, C.POINTER(Share), C.POINTER(Share), C.POINTER(Share)]),
    "spdz_sub_batch": (C.c_int, [vp, C.POINTER(Share), C.POINTER(Share), C.POINTER(Share)]),
    "spdz_mul_mask": (C.c_int, [vp, C.POINTER(Share), C.POINTER(Share), C.POINTER(Triple), vp, vp]),
    "spdz_mul_combine": (C.c_int, [vp, C.POINTER(Triple), vp, vp, C.POINTER(Share)]),
    "spdz_reduce_add": (C.c_int, [vp, C.POINTER(Share), C.POINTER(Share)]),
    "spdz_add_public": (C.c_int, [vp, C.POINTER(Share), vp, C.c_uint64]),
    "spdz_sub_public": (C.c_int, [vp, C.POINTER(Share), vp, C.c_uint64]),
    "spdz_rsub_public": (C.c_int, [vp, C.POINTER(Share), vp, C.c_uint64]),
    "spdz_mul_public": (C.c_int, [vp, C.POINTER(Share), vp, C.c_uint64]),
    "spdz_mul_public_scalar": (C.c_int, [vp, C.POINTER(Share), C.c_uint32]),
    "spdz_share_of_public": (C.c_int, [vp, vp, C.c_uint64, C.POINTER(Share)]),
    "spdz_open_sum": (C.c_int, [vp, vp, C.POINTER(vp), C.c_int, C.c_uint64, vp]),
    "spdz_beaver_open_combine": (C.c_int, [vp, C.POINTER(Triple), vp, C.POINTER(vp), C.c_int, C.POINTER(Share), vp]),
    "spdz_mac_assign_ranks": (C.c_int, [C.POINTER(MacSegment), C.c_uint64]),
    "spdz_mac_sigma": (C.c_int, [vp, C.POINTER(MacSegment), C.c_uint64, C.c_uint64, u32p]),
    "spdz_mac_sigma_records": (C.c_int, [vp, vp, vp, vp, vp, C.c_uint64, C.c_uint64, u32p]),
    "spdz_commit_sigma": (C.c_uint64, [C.c_uint32, C.c_uint64]),
    "spdz_verify_sigmas": (C.c_int, [vp, vp, vp, C.c_uint64]),
    "spdz_fnv1a64": (C.c_uint64, [vp, C.c_uint64, C.c_uint64]),
    "spdz_plan_tiles": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, vp, vp, C.c_uint64, u64p]),
    "spdz_matrix_mask": (C.c_int, [vp, C.POINTER(Share), C.POINTER(Share), C.POINTER(MTriple), vp]),
    "spdz_matrix_open_combine": (C.c_int, [vp, C.POINTER(MTriple), vp, C.POINTER(vp), C.c_int, C.POINTER(Share),
                                           C.POINTER(Share), vp]),
    "spdz_matrix_combine": (C.c_int, [vp, C.POINTER(MTriple), vp, vp, C.POINTER(Share)]),
    "spdz_bmatrix_mask": (C.c_int, [vp, C.POINTER(Share), C.POINTER(Share), C.POINTER(BMTriple), vp]),
    "spdz_bmatrix_open_combine": (C.c_int, [vp, C.POINTER(BMTriple), vp, C.POINTER(vp), C.c_int, C.POINTER(Share),
                                            vp]),
    "spdz_set_gemm_path": (C.c_int, [C.c_int]),
    "spdz_linear_weights_create": (C.c_int, [vp, C.c_uint32, C.c_uint32, vp, C.POINTER(vp)]),
    "spdz_linear_weights_destroy": (C.c_int, [vp]),
    "spdz_linear_secret_public_prepared": (C.c_int, [vp, vp, C.c_uint32, C.POINTER(Share), C.POINTER(Share)]),
    "spdz_linear_secret_public": (C.c_int, [vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, vp, C.POINTER(Share),
                                            C.POINTER(Share), vp, C.POINTER(Share)]),
    "spdz_dealer_alpha": (C.c_int, [C.c_int, C.c_uint64, u32p, u32p]),
    "spdz_dealer_triples": (C.c_int, [vp, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(vp)]),
    "spdz_dealer_share": (C.c_int, [vp, C.c_int, C.c_uint64, C.c_uint64, C.c_uint32, vp, C.c_uint64, vp, vp]),
    "spdz_dealer_matrix_triple": (C.c_int, [vp, C.c_int, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32,
                                            C.c_uint32, C.POINTER(vp), vp]),
    "spdz_dealer_masks": (C.c_int, [vp, C.c_int, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64, vp, vp, vp]),
    "spdz_dealer_draws_triples": (C.c_uint64, [C.c_int, C.c_uint64]),
    "spdz_dealer_draws_share": (C.c_uint64, [C.c_int, C.c_uint64]),
    "spdz_dealer_draws_matrix": (C.c_uint64, [C.c_int, C.c_uint32, C.c_uint32]),
    "spdz_dealer_draws_masks": (C.c_uint64, [C.c_int, C.c_uint64]),
    "spdz_host_add_batch": (C.c_int, [vp, vp, vp, C.c_uint64, vp, vp, C.c_uint64, vp, vp]),
    "spdz_host_sub_batch": (C.c_int, [vp, vp, vp, C.c_uint64, vp, vp, C.c_uint64, vp, vp]),
    "spdz_host_mul_mask": (C.c_int, [vp, vp, vp, C.c_uint64, C.POINTER(vp), C.c_uint64, vp, vp]),
    "spdz_host_mul_combine": (C.c_int, [vp, C.POINTER(vp), C.c_uint64, vp, vp, C.c_uint64, C.c_int, C.c_uint32, vp,
                                        vp]),
    "spdz_host_reduce_add": (C.c_int, [vp, vp, vp, C.c_uint64, vp, vp]),
    "spdz_run_create": (C.c_int, [C.POINTER(Node), C.c_uint32, C.c_uint32, C.c_int, C.POINTER(RunOptions),
                                  C.POINTER(vp)]),
    "spdz_run_destroy": (C.c_int, [vp]),
    "spdz_run_deal": (C.c_int, [vp, C.c_uint64]),
    "spdz_triple_layout": (C.c_int, [C.POINTER(Node), C.c_uint32, C.c_uint64, C.c_uint64, u64p, C.c_uint64, u64p]),
    "spdz_run_load_store": (C.c_int, [vp, C.c_int, C.c_char_p]),
    "spdz_store_inspect": (C.c_int, [C.c_char_p, C.POINTER(StoreInfo)]),
    "spdz_run_bind_input": (C.c_int, [vp, C.c_uint32, vp, C.c_uint64]),
    "spdz_run_share_inputs": (C.c_int, [vp]),
    "spdz_run_online": (C.c_int, [vp, C.c_int, C.POINTER(RunReport)]),
    "spdz_run_outputs": (C.c_int, [vp, vp, C.c_uint64, u64p]),
    "spdz_run_online_begin": (C.c_int, [vp, C.c_int]),
    "spdz_run_output_digest": (C.c_int, [vp, u64p]),
    "spdz_run_mac_check": (C.c_int, [vp, C.c_int, C.c_uint64, C.POINTER(RunReport)]),
    "spdz_run_wait_openings": (C.c_int, [vp]),
    "spdz_run_mac_check_launch": (C.c_int, [vp, C.c_int, C.c_uint64]),
    "spdz_run_set_copy_streams": (C.c_int, [vp, vp, vp]),
    "spdz_run_party_stream": (vp, [vp, C.c_int]),
    "spdz_run_span_ms": (C.c_int, [vp, vp, C.POINTER(C.c_float)]),
    "spdz_run_bind_output": (C.c_int, [vp, vp, C.c_uint64]),
    "spdz_run_node_share": (C.c_int, [vp, C.c_int, C.c_uint32, C.POINTER(Share)]),
    "spdz_run_export": (C.c_int, [vp, vp, C.c_uint64, u64p]),
    "spdz_run_import": (C.c_int, [vp, vp, C.c_uint64]),
    "spdz_run_inject_bitflip": (C.c_int, [vp, C.c_uint32, C.c_int, C.c_int, C.c_uint64, C.c_uint32]),
    "spdz_share_alloc": (C.c_int, [vp, C.c_uint64, C.POINTER(Share)]),
    "spdz_share_free": (C.c_int, [vp, C.POINTER(Share)]),
    "spdz_share_upload": (C.c_int, [vp, C.POINTER(Share), vp, vp, C.c_uint64]),
    "spdz_share_download": (C.c_int, [vp, C.POINTER(Share), vp, vp, C.c_uint64]),
    "spdz_event_record": (C.c_int, [vp, C.POINTER(vp)]),
    "spdz_event_query": (C.c_int, [vp, C.POINTER(C.c_int)]),
    "spdz_event_sync": (C.c_int, [vp]),
    "spdz_event_wait": (C.c_int, [vp, vp]),
    "spdz_event_destroy": (C.c_int, [vp]),
    "spdz_mac_log_append": (C.c_int, [vp, C.c_uint64, vp, vp, vp, C.c_uint64]),
    "spdz_mac_log_size": (C.c_int, [vp, u64p]),
    "spdz_mac_log_sigma": (C.c_int, [vp, C.c_uint64, C.POINTER(C.c_uint32)]),
    "spdz_mac_log_clear": (C.c_int, [vp]),
    "spdz_net_connect": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_char_p), C.c_uint64, C.c_uint64, C.POINTER(vp)]),
    "spdz_net_destroy": (C.c_int, [vp]),
    "spdz_net_send": (C.c_int, [vp, C.c_int, C.c_int, C.c_uint64, vp, C.c_uint32]),
    "spdz_net_recv": (C.c_int, [vp, C.c_int, C.c_int, C.c_uint64, vp, C.c_uint64, u64p]),
    "spdz_net_stats": (C.c_int, [vp, u64p, u64p]),
    "spdz_run_attach_net": (C.c_int, [vp, vp]),
}

_lib = None


def exported_symbols():
    return sorted(_SIGS)


def lib():
    """Load the CUDA back end.  Raises BackendUnavailable if it was never built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise errors.BackendUnavailable(
                f"BackendUnavailable: {LIB_PATH.name} is not built (run __graft_entry__.build()); "
                "there is no CPU fallback")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            if name.startswith("spdz_diag_") and "SPDZ_B200_LIB" in _os.environ and not hasattr(L, name):
                continue  # older variant build under test (experiments only)
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int):
    if rc != 0:
        raise errors.from_code(rc, lib().spdz_last_error().decode(errors="replace"))
