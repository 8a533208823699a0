"""ctypes binding of libhvb200.so (include/hvb200.h).

The shared library is the product: every compute call below runs hand-written
sm_100a kernels. There is no CPU fallback — if the library or a B200 is
missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libhvb200.so"
HEADER = PKG.parent / "include" / "hvb200.h"

HV_OK, HV_ERR_INVALID_ARGUMENT, HV_ERR_DOMAIN, HV_ERR_LOGIC, HV_ERR_CUDA, HV_ERR_NO_DEVICE, HV_ERR_RUNTIME = range(7)
GEN_RANDOM, GEN_SCALE_RANDOM, GEN_SANDWICH = 0, 1, 2
BIND_ID_LEVEL, BIND_PERMUTATION, BIND_APPENDING = 0, 1, 2
METRIC_HAMMING, METRIC_COSINE = 0, 1


class HVError(RuntimeError):
    """Base class; `status` is the hv_status code."""

    status = HV_ERR_RUNTIME


class InvalidArgument(HVError, ValueError):
    """std::invalid_argument in the reference."""

    status = HV_ERR_INVALID_ARGUMENT


class DomainError(HVError, ArithmeticError):
    """std::domain_error in the reference."""

    status = HV_ERR_DOMAIN


class LogicError(HVError):
    status = HV_ERR_LOGIC


class CudaError(HVError):
    status = HV_ERR_CUDA


class NoDevice(HVError):
    status = HV_ERR_NO_DEVICE


_ERRORS = {HV_ERR_INVALID_ARGUMENT: InvalidArgument, HV_ERR_DOMAIN: DomainError, HV_ERR_LOGIC: LogicError,
           HV_ERR_CUDA: CudaError, HV_ERR_NO_DEVICE: NoDevice, HV_ERR_RUNTIME: HVError}


class Model(C.Structure):
    """struct hv_model (model.hpp:22-56 state, caller-owned host arrays)."""

    _fields_ = [("class_count", C.c_size_t), ("dim", C.c_size_t), ("metric", C.c_int), ("gamma", C.c_double),
                ("seed", C.c_uint64), ("accumulators", C.c_void_p), ("class_weight", C.c_void_p),
                ("sample_counts", C.c_void_p), ("class_vectors", C.c_void_p), ("tiebreak", C.c_void_p)]


class EvalReportC(C.Structure):
    """struct hv_eval_report (eval.hpp:13-37)."""

    _fields_ = [("tp", C.c_uint64), ("fp", C.c_uint64), ("tn", C.c_uint64), ("fn", C.c_uint64),
                ("accuracy", C.c_double), ("tpr", C.c_double), ("ppv", C.c_double), ("f1", C.c_double),
                ("has_tpr", C.c_int), ("has_ppv", C.c_int), ("has_f1", C.c_int),
                ("episodes_detected", C.c_uint64), ("episodes_total", C.c_uint64),
                ("episodes_false_positive", C.c_uint64)]


sz, u64, u32, i32, vp, dbl, ci = C.c_size_t, C.c_uint64, C.c_uint32, C.c_int32, C.c_void_p, C.c_double, C.c_int
ST = C.c_int  # hv_status

# name -> (restype, argtypes)
SIGNATURES = {
    "hv_abi_version": (C.c_int, []),
    "hv_last_error": (C.c_char_p, []),
    "hv_words_per_row": (sz, [sz]),
    "hv_kernel_launch_count": (u64, []),
    "hv_context_create": (ST, [ci, C.POINTER(vp)]),
    "hv_context_destroy": (None, [vp]),
    "hv_context_set_stream": (ST, [vp, vp]),
    "hv_context_stream": (vp, [vp]),
    "hv_context_synchronize": (ST, [vp]),
    "hv_splitmix64": (u64, [u64]),
    "hv_derive_seed": (u64, [u64, u64]),
    "hv_generate_random": (ST, [sz, sz, u64, vp]),
    "hv_generate_scale_random": (ST, [sz, sz, u64, vp]),
    "hv_generate_sandwich": (ST, [sz, sz, u64, vp]),
    "hv_make_codebook": (ST, [ci, sz, sz, sz, u64, vp, vp]),
    "hv_pack": (ST, [vp, vp, sz, sz, vp]),
    "hv_unpack": (ST, [vp, vp, sz, sz, vp]),
    "hv_xor_bind": (ST, [vp, vp, sz, sz, vp, sz, sz, vp]),
    "hv_rotate": (ST, [vp, vp, sz, sz, sz, vp]),
    "hv_horizontal_sum": (ST, [vp, vp, sz, sz, vp]),
    "hv_transpose": (ST, [vp, vp, sz, sz, vp]),
    "hv_vertical_sum": (ST, [vp, vp, sz, sz, vp]),
    "hv_majority_binarize": (ST, [vp, vp, sz, u64, vp, sz, sz, vp]),
    "hv_fit_discretizer": (ST, [vp, vp, sz, sz, sz, vp, vp]),
    "hv_discretize_matrix": (ST, [vp, vp, sz, sz, vp, vp, sz, vp]),
    "hv_encode_batch": (ST, [vp, vp, sz, sz, vp, vp, sz, sz, ci, vp, sz, sz, vp]),
    "hv_make_empty_model": (ST, [C.POINTER(Model)]),
    "hv_refresh_binarization": (ST, [vp, C.POINTER(Model), sz]),
    "hv_train_classical": (ST, [vp, vp, sz, sz, vp, sz, C.POINTER(Model)]),
    "hv_online_update": (ST, [vp, C.POINTER(Model), vp, sz, sz, vp, sz, vp, vp]),
    "hv_train_online": (ST, [vp, vp, sz, sz, vp, sz, sz, C.POINTER(Model)]),
    "hv_predict": (ST, [vp, C.POINTER(Model), vp, sz, sz, vp, vp]),
    "hv_hamming_distance_words": (dbl, [vp, vp, sz]),
    "hv_hamming_distance": (ST, [vp, vp, vp, sz, C.POINTER(dbl)]),
    "hv_cosine_similarity": (ST, [vp, vp, sz, vp, sz, C.POINTER(dbl)]),
    "hv_host_narrow_bins": (ST, [vp, sz, sz, sz, vp, sz, C.POINTER(u64)]),
    "hv_dev_check": (ST, [vp]),
    "hv_dev_narrow_bins": (ST, [vp, vp, sz, sz, sz, vp, sz]),
    "hv_dev_encode": (ST, [vp, vp, sz, sz, sz, vp, vp, sz, sz, ci, vp, vp]),
    "hv_dev_class_counts": (ST, [vp, vp, sz, sz, vp, sz, vp, vp]),
    "hv_dev_binarize_counts": (ST, [vp, vp, vp, sz, sz, vp, vp]),
    "hv_dev_predict_hamming": (ST, [vp, vp, sz, sz, vp, sz, vp, vp, vp]),
    "hv_dev_train_online": (ST, [vp, vp, sz, sz, vp, sz, sz, dbl, vp, vp, vp, vp, vp]),
    "hv_dev_online_delta": (ST, [vp, vp, sz, sz, vp, sz, vp, dbl, vp, vp, vp, vp]),
    "hv_dev_apply_online_delta": (ST, [vp, sz, sz, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "hv_dev_synth": (ST, [vp, u64, sz, sz, sz, sz, ci, u64, vp, sz, vp]),
    "hv_dev_encode_words": (ST, [vp, vp, sz, sz, sz, vp, vp, sz, sz, ci, vp, sz, sz, vp, sz]),
    "hv_dev_online_slice_init": (ST, [vp, vp, sz, vp, sz, sz, sz, sz, vp, vp, vp, vp, vp]),
    "hv_dev_online_partial_popc": (ST, [vp, vp, sz, sz, vp, sz, vp]),
    "hv_dev_online_partial_popc_peers": (ST, [vp, vp, sz, sz, vp, sz, vp, sz]),
    "hv_dev_online_slice_update": (ST, [vp, vp, sz, sz, sz, sz, vp, sz, vp, dbl, vp, vp, vp, vp, vp]),
    "hv_dev_online_sliced_run_peers": (ST, [vp, vp, sz, sz, sz, sz, vp, sz, sz, dbl, vp, vp, vp, vp, vp, vp, vp, sz,
                                            sz, u32, vp, vp, vp, vp]),
    "hv_shared_handle_size": (sz, []),
    "hv_shared_alloc": (ST, [vp, sz, C.POINTER(vp), vp]),
    "hv_shared_open": (ST, [vp, vp, C.POINTER(vp)]),
    "hv_shared_close": (ST, [vp, vp]),
    "hv_shared_free": (ST, [vp, vp]),
    "hv_dev_class_counts_peers": (ST, [vp, vp, sz, sz, vp, sz, vp, vp, sz]),
    "hv_dev_class_counts_peers_pitched": (ST, [vp, vp, sz, sz, sz, vp, sz, vp, vp, sz]),
    "hv_row_pitch_words": (sz, [sz]),
    "hv_dev_class_counts_pitched": (ST, [vp, vp, sz, sz, sz, vp, sz, vp, vp]),
    "hv_dev_predict_hamming_pitched": (ST, [vp, vp, sz, sz, vp, sz, sz, vp, vp, vp]),
    "hv_dev_signal_peers": (ST, [vp, vp, sz, sz, u32]),
    "hv_dev_wait_peers": (ST, [vp, vp, sz, u32]),
    "hv_dataset_create": (ST, [vp, vp, sz, sz, vp, C.POINTER(vp)]),
    "hv_dataset_destroy": (None, [vp]),
    "hv_dataset_fold": (ST, [vp, vp, vp, sz, vp, sz, sz, vp, vp, sz, ci, vp, sz, ci, dbl, vp, ci, sz, vp, vp, vp]),
    "hv_smooth_labels": (ST, [vp, vp, sz, sz, vp]),
    "hv_sample_metrics": (ST, [vp, vp, sz, vp, sz, ci, vp]),
    "hv_episode_metrics": (ST, [vp, vp, sz, vp, sz, ci, vp, vp, vp]),
    "hv_dev_smooth_labels": (ST, [vp, vp, sz, sz, vp]),
    "hv_dev_eval_counts": (ST, [vp, vp, vp, sz, ci, vp, vp]),
    "hv_experiment_create": (ST, [vp, vp, C.POINTER(vp)]),
    "hv_experiment_destroy": (None, [vp]),
    "hv_experiment_fold": (ST, [vp, vp, vp, sz, vp, sz, sz, vp, vp, sz, ci, vp, sz, ci, dbl, vp, ci, sz]),
    "hv_experiment_finish": (ST, [vp, vp, sz, sz, ci, vp, vp, vp, vp, vp, vp]),
    "hv_fold_encode_train": (ST, [vp, vp, sz, vp, vp, sz, sz, vp, vp, sz, sz, vp, sz, C.POINTER(vp)]),
    "hv_fold_counts": (ST, [vp, C.POINTER(vp), C.POINTER(vp)]),
    "hv_fold_predict": (ST, [vp, vp, vp, vp]),
    "hv_fold_destroy": (None, [vp]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load libhvb200.so (building it first if this checkout has none)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    from . import _build

                    _build.build()
                L = C.CDLL(str(LIB_PATH))
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = L
    return _lib


def check(status: int) -> None:
    if status != HV_OK:
        msg = lib().hv_last_error()
        msg = msg.decode() if msg else ""
        raise _ERRORS.get(status, HVError)(msg)


class Context:
    """Owns an hv_context (one CUDA device, one stream pair)."""

    def __init__(self, device: int = 0):
        h = vp()
        check(lib().hv_context_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    def set_stream(self, stream_ptr: int | None):
        check(lib().hv_context_set_stream(self.handle, stream_ptr))

    def synchronize(self):
        check(lib().hv_context_synchronize(self.handle))

    def dev_check(self):
        check(lib().hv_dev_check(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            lib().hv_context_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_contexts: dict[int, Context] = {}


def context(device: int = 0) -> Context:
    ctx = _contexts.get(device)
    if ctx is None:
        ctx = _contexts[device] = Context(device)
    return ctx


def launch_count() -> int:
    return int(lib().hv_kernel_launch_count())
