"""ctypes binding of ``libcovap_b200.so`` (the C-ABI in ``include/covap_c.h``).

This is the reference-side binding a Python caller (a DDP comm hook, the
bench, the tests) uses.  There is no fallback: if the shared library is
missing the import fails loudly, and every device entry point returns
``COVAP_ERR_NO_DEVICE`` rather than computing on the CPU.
"""
import ctypes
import os

from .errors import raise_for_status

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcovap_b200.so")
# Development override (scripts/variants.sh builds kernel variants elsewhere).
LIB_PATH = os.environ.get("COVAP_LIB_PATH", LIB_PATH)

u8p = ctypes.POINTER(ctypes.c_uint8)
u32p = ctypes.POINTER(ctypes.c_uint32)
u64p = ctypes.POINTER(ctypes.c_uint64)
f64p = ctypes.POINTER(ctypes.c_double)
vp = ctypes.c_void_p
sz = ctypes.c_size_t
i32 = ctypes.c_int
u32 = ctypes.c_uint32
u64 = ctypes.c_uint64
f64 = ctypes.c_double

F32, F64 = 0, 1


class EfC(ctypes.Structure):
    _fields_ = [("enabled", i32), ("init_value", f64), ("ascend_steps", u64),
                ("ascend_range", f64)]


class PlanInfoC(ctypes.Structure):
    _fields_ = [("n_layers", u64), ("n_buckets", u64), ("n_tensors", u64), ("total_numel", u64),
                ("twice_median", u64), ("interval", u32), ("rule", ctypes.c_int32),
                ("sharded", ctypes.c_int32), ("align", ctypes.c_int32),
                ("max_send_elems", u64), ("device_numel", u64), ("padded", ctypes.c_int32)]


class BucketRangeC(ctypes.Structure):
    _fields_ = [("bucket_begin", u64), ("bucket_end", u64), ("sel_begin", u64),
                ("sel_end", u64), ("send_offset", u64), ("device_begin", u64)]


class SettingsC(ctypes.Structure):
    _fields_ = [("interval", u32), ("auto_interval", ctypes.c_int32), ("rule", ctypes.c_int32),
                ("ef", EfC)]


class CcrResultC(ctypes.Structure):
    _fields_ = [("ccr", f64), ("comp_ms", f64), ("comm_aligned_ms", f64),
                ("recommended_interval", u32)]


class FilterC(ctypes.Structure):
    _fields_ = [("kind", i32), ("interval", u32), ("rule", i32), ("k_fraction", f64),
                ("seed", u64)]


# name -> (restype, argtypes); restype None means covap_status (int) checked.
_SIGS = {
    "covap_last_error": (ctypes.c_char_p, []),
    "covap_version": (i32, []),
    "covap_device_count": (None, [ctypes.POINTER(i32)]),
    "covap_plan_create": (None, [u64p, u32p, sz, u64, u32, i32, i32, ctypes.POINTER(vp)]),
    "covap_plan_create_ex": (None, [u64p, u32p, sz, u64, u32, i32, i32, i32, ctypes.POINTER(vp)]),
    "covap_plan_destroy": ("void", [vp]),
    "covap_plan_get_info": (None, [vp, ctypes.POINTER(PlanInfoC)]),
    "covap_plan_buckets": (None, [vp, u64p, u64p, u64p, u64p]),
    "covap_plan_tensors": (None, [vp, u64p, u64p, u64p]),
    "covap_plan_selection": (None, [vp, u64, u8p]),
    "covap_plan_bucket_range": (None, [vp, u64, sz, ctypes.POINTER(BucketRangeC)]),
    "covap_plan_send_elems": (None, [vp, u64, u64p, u64p]),
    "covap_median_twice": (None, [u64p, sz, u64p]),
    "covap_select_tensors": (None, [u64, u32, sz, i32, u8p]),
    "covap_ef_coefficient": (None, [u64, ctypes.POINTER(EfC), f64p]),
    "covap_ccr": (None, [f64, f64, f64p]),
    "covap_choose_interval": (None, [f64, u32p]),
    "covap_profile_ccr": (None, [f64p, f64p, sz, sz, sz, f64, f64p, f64p, f64p, u32p]),
    "covap_state_create": (None, [vp, i32, i32, ctypes.POINTER(EfC), ctypes.POINTER(vp)]),
    "covap_state_destroy": ("void", [vp]),
    "covap_state_residual": (None, [vp, ctypes.POINTER(vp), u64p]),
    "covap_state_send": (None, [vp, ctypes.POINTER(vp), u64p]),
    "covap_state_get_step": (None, [vp, u64p]),
    "covap_state_set_step": (None, [vp, u64]),
    "covap_state_set_fused": (None, [vp, i32]),
    "covap_state_set_host_ramp": (None, [vp, u64]),
    "covap_state_set_pipeline": (None, [vp, i32]),
    "covap_state_reset": (None, [vp, vp]),
    "covap_filter_pack": (None, [vp, vp, vp, sz, sz, vp]),
    "covap_filter_pack_zero": (None, [vp, vp, vp, vp, sz, sz, vp]),
    "covap_unpack_selected": (None, [vp, vp, vp, f64, sz, sz, vp]),
    "covap_unpack": (None, [vp, vp, vp, f64, i32, sz, sz, vp]),
    "covap_filter_unpack": (None, [vp, vp, vp, f64, sz, sz, vp]),
    "covap_filter_sgd": (None, [vp, vp, vp, f64, f64, sz, sz, vp]),
    "covap_unpack_sgd": (None, [vp, vp, vp, f64, f64, i32, sz, sz, vp]),
    "covap_sync_step_sgd": (None, [vp, vp, vp, vp, f64, vp]),
    "covap_step_end": (None, [vp]),
    "covap_sync_step": (None, [vp, vp, vp, vp, vp]),
    "covap_sync_step_host": (None, [vp, vp, vp, vp, vp, vp, u64, vp]),
    "covap_bucket_ready": (None, [vp, vp, sz, vp, vp, vp]),
    "covap_step_finish": (None, [vp, vp]),
    "covap_bucket_ready_local": (None, [vp, vp, sz, vp, vp, vp]),
    "covap_dense_bucket_ready_local": (None, [vp, vp, sz, vp, vp, vp]),
    "covap_dense_bucket_ready": (None, [vp, vp, sz, vp, vp, vp]),
    "covap_state_last_comm_ms": (None, [vp, f64p, sz]),
    "covap_state_set_timeline": (None, [vp, i32]),
    "covap_state_timeline": (None, [vp, f64p, sz]),
    "covap_overlap_schedule": (None, [f64, f64p, f64p, f64p, u8p, sz, f64p, f64p, f64p, f64p, f64p,
                                      ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(sz),
                                      ctypes.POINTER(ctypes.c_int64), f64p, ctypes.POINTER(sz)]),
    "covap_comm_unique_id": (None, [ctypes.c_char_p]),
    "covap_comm_create": (None, [ctypes.c_char_p, i32, i32, i32, ctypes.POINTER(vp)]),
    "covap_comm_destroy": ("void", [vp]),
    "covap_comm_size": (None, [vp, ctypes.POINTER(i32), ctypes.POINTER(i32)]),
    "covap_allreduce": (None, [vp, vp, u64, i32, vp]),
    "covap_state_use_symmetric": (None, [vp, vp]),
    "covap_comm_allreduce_mean": (None, [vp, i32, vp, vp, u64, vp]),
    "covap_comm_profile_exchange": (None, [vp, f64p, sz, f64, f64p, f64p]),
    "covap_settings_default": (None, [ctypes.POINTER(SettingsC)]),
    "covap_settings_from_json": (None, [ctypes.c_char_p, ctypes.POINTER(SettingsC)]),
    "covap_resolve_interval": (None, [ctypes.POINTER(SettingsC), f64, ctypes.POINTER(u32)]),
    "covap_ccr_decide": (None, [vp, f64p, sz, f64, ctypes.POINTER(CcrResultC)]),
    "covap_peer_create": (None, [vp, i32, i32, ctypes.POINTER(vp)]),
    "covap_peer_destroy": ("void", [vp]),
    "covap_peer_export": (None, [vp, ctypes.c_char_p, sz, ctypes.POINTER(sz)]),
    "covap_peer_import": (None, [vp, ctypes.c_char_p, sz]),
    "covap_peer_attach_local": (None, [ctypes.POINTER(vp), i32]),
    "covap_peer_create_nccl": (None, [vp, vp, i32, ctypes.POINTER(vp)]),
    "covap_state_side_stream": (None, [vp, ctypes.POINTER(vp)]),
    "covap_state_set_free_sms": (None, [vp, i32]),
    "covap_peer_multimem": (None, [vp, ctypes.POINTER(i32)]),
    "covap_peer_set_limits": (None, [vp, i32, f64]),
    "covap_peer_set_fused": (None, [vp, i32]),
    "covap_peer_check": (None, [vp]),
    "covap_peer_sync_step": (None, [vp, vp, vp, vp, vp]),
    "covap_device_alloc": (None, [i32, u64, ctypes.POINTER(vp)]),
    "covap_device_free": (None, [i32, vp]),
    "covap_memcpy": (None, [vp, vp, u64, i32, vp]),
    "covap_stream_synchronize": (None, [vp]),
    "covap_embed": (None, [i32, i32, vp, vp, u64, u64p, u64p, u64p, sz, f64, i32, vp]),
    "covap_mean_rows": (None, [i32, i32, vp, vp, u64, u64, vp]),
    # baseline compressors under error feedback
    "covap_feedback_create": (None, [u64p, sz, i32, ctypes.POINTER(EfC), ctypes.POINTER(FilterC),
                                     i32, ctypes.POINTER(vp)]),
    "covap_feedback_destroy": ("void", [vp]),
    "covap_feedback_residual": (None, [vp, ctypes.POINTER(vp), u64p]),
    "covap_feedback_get_step": (None, [vp, u64p]),
    "covap_feedback_set_step": (None, [vp, u64]),
    "covap_feedback_reset": (None, [vp, vp]),
    "covap_feedback_step": (None, [vp, vp, vp, vp]),
    "covap_feedback_transmitted": (None, [vp, u64, u64p, u64p]),
    "covap_feedback_saturations": (None, [vp, u64p, vp]),
    "covap_feedback_sync_step": (None, [vp, vp, vp, vp, vp]),
    "covap_feedback_pack": (None, [vp, vp, vp, vp]),
    "covap_feedback_wire": (None, [vp, ctypes.POINTER(vp), u64p, ctypes.POINTER(vp), u64p]),
    "covap_feedback_combine": (None, [vp, vp, vp, i32, vp, vp]),
    "covap_sparsifier_k": (None, [u64, f64, u64p]),
    "covap_topk_compress": (None, [i32, i32, vp, u64, f64, vp, vp, u64p, vp]),
    "covap_randomk_compress": (None, [i32, i32, vp, u64, f64, u64, vp, vp, u64p, vp]),
    "covap_fp16_roundtrip": (None, [i32, i32, vp, u64, vp, u64p, vp]),
    "covap_fp16_encode": (None, [i32, i32, vp, u64, vp, u64p, vp]),
    "covap_fp16_decode": (None, [i32, vp, u64, vp, vp]),
    "covap_stream_key": (u64, [u64, u64, u64]),
    "covap_generate": (None, [vp, u64, i32, u64, i32, u64, vp]),
    "covap_spin": (None, [f64, i32, vp]),
    "covap_busy": (None, [ctypes.c_double, ctypes.c_double, vp]),
}

EXPORTED = tuple(_SIGS)


class _Lib:
    def __init__(self, path=LIB_PATH):
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (make -C paper_2311_04499_b200/csrc). There is no CPU fallback.")
        self.path = path
        self.dll = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(self.dll, name)
            fn.argtypes = args
            if res is None:
                fn.restype = ctypes.c_int
            elif res == "void":
                fn.restype = None
            else:
                fn.restype = res
            if res is None:
                setattr(self, name, self._checked(fn))
            else:
                setattr(self, name, fn)

    def _checked(self, fn):
        dll = self.dll

        def call(*args):
            st = fn(*args)
            if st:
                raise_for_status(st, dll.covap_last_error().decode(errors="replace"))
            return st
        call.__name__ = fn.__name__
        return call


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        _LIB = _Lib()
    return _LIB
