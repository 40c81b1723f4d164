"""ctypes binding of libturnstile_b200.so (the C ABI in include/turnstile_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_1912_11554_b200/csrc``).  There is no CPU fallback: if the
library or a CUDA device is missing, every device entry point raises
``RuntimeError`` immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libturnstile_b200.so")

TS_OK, TS_EINVAL, TS_ECUDA, TS_EUNSUPPORTED = 0, 1, 2, 3
TS_STD_NORMAL, TS_GAUSSIAN, TS_LOGISTIC, TS_FUNNEL, TS_EIGHT_SCHOOLS, TS_DENSE_GAUSS = 0, 1, 2, 3, 4, 5
TS_PREC_FP64, TS_PREC_FP32, TS_PREC_TF32, TS_PREC_FP64X = 0, 1, 2, 3
TS_GENERALIZED, TS_CLASSIC = 0, 1
TS_EXEC_THREAD, TS_EXEC_BLOCK, TS_EXEC_WARP = 0, 1, 2
TS_STATUS_SYNC_TIMEOUT = 2
ABI_VERSION = 1

# every symbol include/turnstile_b200.h declares
EXPORTS = (
    "ts_last_error",
    "ts_abi_version",
    "ts_model_create",
    "ts_model_destroy",
    "ts_model_dim",
    "ts_model_set_grid",
    "ts_potential_grad",
    "ts_eval_bench",
    "ts_leapfrog",
    "ts_build_tree",
    "ts_transition",
    "ts_find_step_size",
    "ts_run_chains",
    "ts_rng_probe",
    "ts_libm_probe",
    "ts_dense_transform",
    "ts_peer_mailbox_create",
    "ts_peer_mailbox_connect",
    "ts_logistic_partial_sums",
    "ts_gemm_tf32_probe",
    "ts_hmc_transition",
    "ts_model_set_virtual_ranks",
    "ts_pooled_covariance",
    "ts_pooled_covariance_workspace",
    "ts_model_error",
    "ts_chain_diagnostics",
    "ts_chain_diagnostics_workspace",
)


class SamplerCfgC(ctypes.Structure):
    _fields_ = [
        ("step_size", ctypes.c_double),
        ("max_tree_depth", ctypes.c_int32),
        ("criterion", ctypes.c_int32),
        ("divergence_threshold", ctypes.c_double),
    ]


class RunCfgC(ctypes.Structure):
    _fields_ = [
        ("num_warmup", ctypes.c_int32),
        ("num_samples", ctypes.c_int32),
        ("target_accept", ctypes.c_double),
        ("has_sampler", ctypes.c_int32),
        ("keep_warmup", ctypes.c_int32),
        ("sampler", SamplerCfgC),
    ]


_lib = None
_lock = threading.Lock()

_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_U64 = ctypes.c_uint64
_I64 = ctypes.c_int64


def _declare(lib):
    lib.ts_last_error.restype = ctypes.c_char_p
    lib.ts_last_error.argtypes = []
    lib.ts_abi_version.restype = _I
    lib.ts_model_create.argtypes = [_I, _I, _P, _I, _P, _P, _I64, _I, _I, ctypes.POINTER(_P)]
    lib.ts_model_destroy.argtypes = [_P]
    lib.ts_model_dim.argtypes = [_P]
    lib.ts_model_set_grid.argtypes = [_P, _I]
    lib.ts_potential_grad.argtypes = [_P, _P, _I, _P, _P]
    lib.ts_eval_bench.argtypes = [_P, _P, _I, _P, _P]
    lib.ts_leapfrog.argtypes = [_P, _P, _P, _D, _P, _I, _P]
    lib.ts_build_tree.argtypes = [_P, ctypes.POINTER(SamplerCfgC), _P, _P, _I, _D, _D, _U64, _U64, _P, _P, _I, _P, _I,
                                  _P, _I, _P]
    lib.ts_transition.argtypes = [_P, ctypes.POINTER(SamplerCfgC), _P, _P, _P, _U64, _U64, _P, _P, _I, _P, _I, _P]
    lib.ts_find_step_size.argtypes = [_P, _P, _P, _P, _U64, _U64, _D, _P, _I, _P]
    lib.ts_run_chains.argtypes = [_P, ctypes.POINTER(RunCfgC), _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P]
    lib.ts_rng_probe.argtypes = [_U64, _U64, _I, _I, _P, _P]
    lib.ts_libm_probe.argtypes = [_I, _P, _P, ctypes.c_int64, _P]
    lib.ts_dense_transform.argtypes = [_P, _P, _P, ctypes.c_int64, _I, _P]
    lib.ts_peer_mailbox_create.argtypes = [_P, _I, _I, _P]
    lib.ts_peer_mailbox_connect.argtypes = [_P, _P]
    lib.ts_logistic_partial_sums.argtypes = [_P, _P, _P, _P]
    lib.ts_gemm_tf32_probe.argtypes = [_P, _P, _P, _I, _I, _I, _I, _P]
    lib.ts_hmc_transition.argtypes = [_P, ctypes.POINTER(SamplerCfgC), _P, _P, _P, _U64, _U64, _I, _P, _I, _P]
    lib.ts_model_set_virtual_ranks.argtypes = [_P, _I]
    lib.ts_pooled_covariance.argtypes = [_P, ctypes.c_int64, _I, _I, _P, _P, _P, _P]
    lib.ts_pooled_covariance_workspace.argtypes = [ctypes.c_int64, _I]
    lib.ts_model_error.argtypes = [_P, ctypes.POINTER(_I)]
    lib.ts_chain_diagnostics.argtypes = [_P, _I, _I, _I, _P, _P, _P, _P]
    lib.ts_chain_diagnostics_workspace.argtypes = [_I, _I, _I]
    for name in EXPORTS:
        if name not in ("ts_last_error",):
            getattr(lib, name).restype = _I
    lib.ts_pooled_covariance_workspace.restype = ctypes.c_int64
    lib.ts_chain_diagnostics_workspace.restype = ctypes.c_int64


def load_library(path: str = LIB_PATH):
    """Load (once) and return the ctypes handle; raises RuntimeError if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RuntimeError(
                    f"CUDA extension {path} is missing; run __graft_entry__.build() "
                    "(no CPU fallback exists by design)"
                )
            lib = ctypes.CDLL(path)
            _declare(lib)
            if lib.ts_abi_version() != ABI_VERSION:
                raise RuntimeError("libturnstile_b200.so ABI version mismatch")
            _lib = lib
        return _lib


def check(code: int) -> None:
    if code == TS_OK:
        return
    msg = load_library().ts_last_error().decode(errors="replace")
    if code == TS_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


SYNC_TIMEOUT_MSG = ("a device synchronisation wait (grid barrier / peer mailbox / served flag) exceeded "
                    "TS_SPIN_TIMEOUT_S; the kernel gave up instead of hanging and the model is poisoned")


def check_model(handle) -> None:
    """Raise RuntimeError if a persistent kernel on this model gave up on a
    wait (sticky device error word, ts_model_error; synchronises)."""
    lib = load_library()
    code = _I(0)
    check(lib.ts_model_error(handle, ctypes.byref(code)))
    if code.value:
        raise RuntimeError(SYNC_TIMEOUT_MSG)


def check_spec(spec, handle) -> None:
    """check_model for the models whose kernels wait across CTAs/GPUs."""
    if spec.kind in (TS_LOGISTIC, TS_DENSE_GAUSS):
        check_model(handle)


def torch_cuda():
    """torch with a usable CUDA device, or RuntimeError (no CPU fallback)."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_1912_11554_b200 requires a CUDA device (B200); none is available")
    return torch


def ptr(t) -> int:
    return t.data_ptr() if t is not None else 0


def stream_ptr(torch, device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def to_dev_f64(torch, arr, device):
    return torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float64)).to(device)


def cuda_device(torch, device=None):
    """Normalise ``device`` (None, int, str, torch.device) to torch.device('cuda', i)."""
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device) if not isinstance(device, int) else torch.device("cuda", device)
    if d.type != "cuda":
        raise ValueError("device must be a CUDA device")
    return torch.device("cuda", d.index if d.index is not None else torch.cuda.current_device())
