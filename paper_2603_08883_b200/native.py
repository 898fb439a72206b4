"""ctypes binding of the engine's C-ABI (include/iqcc_b200.h).

The engine is ``paper_2603_08883_b200/libiqcc_b200.so`` built in-tree from
``csrc/`` for sm_100a.  There is no CPU fallback: if the library cannot be
loaded (or built with ``make -C paper_2603_08883_b200/csrc``) importing this
module raises ``ImportError``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IQCC_LIB") or os.path.join(HERE, "libiqcc_b200.so")  # IQCC_LIB: tuning builds
CSRC = os.path.join(HERE, "csrc")

IQCC_OK, IQCC_EINVAL, IQCC_ERUNTIME, IQCC_ECUDA, IQCC_ENOMEM = 0, 1, 2, 3, 4


def build(force: bool = False) -> str:
    """Compile the engine with nvcc (sm_100a) into LIB_PATH."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-j8", "-C", CSRC], check=True)
    return LIB_PATH


class DressStats(C.Structure):
    _fields_ = [("n_in", C.c_size_t), ("n_anticommuting", C.c_size_t), ("n_out", C.c_size_t)]


class CompressStatsC(C.Structure):
    _fields_ = [("dropped_terms", C.c_size_t), ("dropped_weight", C.c_double)]


class ExchangeStats(C.Structure):
    _fields_ = [("mask", C.c_size_t), ("sent_terms", C.c_size_t), ("recv_terms", C.c_size_t),
                ("bytes_wire", C.c_size_t), ("bytes_reference", C.c_size_t)]


class MessageRecord(C.Structure):
    """iqcc_message_record = MessageRecord (iqcc/partition.hpp:135-140)."""
    _fields_ = [("source", C.c_size_t), ("destination", C.c_size_t), ("terms", C.c_size_t),
                ("bytes", C.c_size_t)]


_vp = C.c_void_p
_u64p = C.c_void_p  # raw addresses (numpy .ctypes.data or device pointers)
_f64p = C.c_void_p
_szp = C.c_void_p

_SIGS = {
    "iqcc_gpu_last_error": (C.c_char_p, []),
    "iqcc_gpu_init": (C.c_int, [C.c_int]),
    "iqcc_gpu_set_stream": (C.c_int, [_vp]),
    "iqcc_gpu_finalize": (C.c_int, []),
    "iqcc_gpu_launch_count": (C.c_uint64, []),
    "iqcc_gpu_profile_enable": (C.c_int, [C.c_int]),
    "iqcc_gpu_profile_get": (C.c_int, [C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]),
    "iqcc_gpu_profile_reset": (C.c_int, []),
    "iqcc_gpu_profile_bytes": (C.c_int, [C.c_char_p, C.POINTER(C.c_double)]),
    "iqcc_gpu_sum_create": (C.c_int, [C.c_size_t, _u64p, _f64p, C.c_size_t, C.POINTER(_vp)]),
    "iqcc_gpu_sum_create_device": (C.c_int, [C.c_size_t, _u64p, _f64p, C.c_size_t, C.POINTER(_vp)]),
    "iqcc_gpu_sum_generate_mol": (C.c_int, [C.c_size_t, C.c_size_t, C.c_uint64, C.POINTER(_vp)]),
    "iqcc_gpu_sum_clone": (C.c_int, [_vp, C.POINTER(_vp)]),
    "iqcc_gpu_read_pauli_file": (C.c_int, [C.c_char_p, C.POINTER(_vp)]),
    "iqcc_gpu_write_pauli_file": (C.c_int, [_vp, C.c_char_p]),
    "iqcc_gpu_jordan_wigner_fcidump": (C.c_int, [C.c_char_p, C.POINTER(C.c_size_t), C.POINTER(_vp)]),
    "iqcc_gpu_sum_destroy": (C.c_int, [_vp]),
    "iqcc_gpu_sum_qubits": (C.c_int, [_vp, C.POINTER(C.c_size_t)]),
    "iqcc_gpu_sum_size": (C.c_int, [_vp, C.POINTER(C.c_size_t)]),
    "iqcc_gpu_sum_download": (C.c_int, [_vp, _u64p, _f64p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "iqcc_gpu_sum_download_device": (C.c_int, [_vp, _u64p, _f64p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "iqcc_gpu_sum_raw": (C.c_int, [_vp, _u64p, _f64p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "iqcc_gpu_dress": (C.c_int, [_vp, _u64p, C.c_double, C.c_double, C.c_double, C.POINTER(DressStats)]),
    "iqcc_gpu_compress": (C.c_int, [_vp, C.c_double, C.c_size_t, C.POINTER(CompressStatsC)]),
    "iqcc_gpu_dress_sequence": (C.c_int, [_vp, C.c_size_t, _u64p, _f64p, _f64p, C.c_double, C.c_size_t,
                                          C.c_double, C.POINTER(CompressStatsC), C.POINTER(C.c_size_t)]),
    "iqcc_gpu_growth_split": (C.c_int, [_vp, _u64p, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "iqcc_gpu_sortless_stats": (C.c_int, [_vp, _u64p, C.c_double, C.POINTER(C.c_size_t),
                                          C.POINTER(C.c_size_t)]),
    "iqcc_gpu_expect": (C.c_int, [_vp, _f64p, C.POINTER(C.c_double)]),
    "iqcc_gpu_qmf_energy_gradient": (C.c_int, [_vp, _f64p, _f64p, C.POINTER(C.c_double), _f64p]),
    "iqcc_gpu_qcc_energy": (C.c_int, [_vp, C.c_size_t, _u64p, _f64p, _f64p, _f64p, C.POINTER(C.c_double)]),
    "iqcc_gpu_qcc_gradient": (C.c_int, [_vp, C.c_size_t, _u64p, _f64p, _f64p, _f64p, _f64p]),
    "iqcc_gpu_gradients": (C.c_int, [_vp, _f64p, _u64p, C.c_size_t, C.c_int, _f64p]),
    "iqcc_gpu_poly_kernels": (C.c_int, [_vp, _f64p, C.c_int, _u64p, C.c_size_t, _f64p, _f64p]),
    "iqcc_gpu_parallel_poly_kernels": (C.c_int, [_vp, _f64p, C.c_int, _u64p, C.c_size_t, _f64p, _f64p]),
    "iqcc_gpu_dis_candidates": (C.c_int, [_vp, _f64p, C.c_int, C.c_size_t, C.c_double, C.c_size_t, C.c_int,
                                          C.c_uint64, _u64p, _f64p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "iqcc_gpu_choose_partition_bits": (C.c_int, [_vp, C.c_size_t, _szp, C.POINTER(C.c_double)]),
    "iqcc_gpu_sum_restrict": (C.c_int, [_vp, C.c_size_t, _szp, _szp, C.c_int]),
    "iqcc_gpu_nccl_unique_id": (C.c_int, [_vp]),
    "iqcc_gpu_comm_init": (C.c_int, [_vp, C.c_int, C.c_int]),
    "iqcc_gpu_comm_destroy": (C.c_int, []),
    "iqcc_gpu_parallel_dress": (C.c_int, [_vp, C.c_size_t, _szp, _szp, _u64p, C.c_double, C.c_double,
                                          C.c_double, C.c_size_t, C.POINTER(ExchangeStats),
                                          C.POINTER(CompressStatsC)]),
    "iqcc_gpu_parallel_dress_sequence": (C.c_int, [_vp, C.c_size_t, _szp, _szp, C.c_size_t, _u64p, _f64p,
                                                   _f64p, C.c_double, C.c_size_t, C.POINTER(ExchangeStats),
                                                   C.POINTER(CompressStatsC), C.POINTER(C.c_size_t)]),
    "iqcc_gpu_parallel_expect": (C.c_int, [_vp, _f64p, C.POINTER(C.c_double)]),
    "iqcc_gpu_parallel_compress": (C.c_int, [_vp, C.c_double, C.c_size_t, C.POINTER(CompressStatsC)]),
    "iqcc_gpu_parallel_reserve": (C.c_int, [_vp, C.c_size_t]),
    "iqcc_gpu_parallel_size": (C.c_int, [_vp, C.POINTER(C.c_size_t)]),
    "iqcc_gpu_parallel_qmf_energy_gradient": (C.c_int, [_vp, _f64p, _f64p, C.POINTER(C.c_double), _f64p]),
    "iqcc_gpu_parallel_gradients": (C.c_int, [_vp, _f64p, _u64p, C.c_size_t, C.c_int, _f64p]),
    "iqcc_gpu_merge_sums": (C.c_int, [_vp, _vp, C.c_double, C.POINTER(_vp)]),
    "iqcc_gpu_psum_distribute": (C.c_int, [C.c_size_t, _u64p, _f64p, C.c_size_t, C.c_size_t, _szp, _szp,
                                           C.c_size_t, _vp, C.POINTER(_vp)]),
    "iqcc_gpu_psum_create_shards": (C.c_int, [C.c_size_t, C.c_size_t, _szp, _szp, C.c_size_t, _vp, _vp, _vp,
                                              _szp, C.POINTER(_vp)]),
    "iqcc_gpu_psum_destroy": (C.c_int, [_vp]),
    "iqcc_gpu_psum_info": (C.c_int, [_vp, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "iqcc_gpu_psum_shard_sizes": (C.c_int, [_vp, _szp]),
    "iqcc_gpu_psum_owner": (C.c_int, [_vp, _szp]),
    "iqcc_gpu_psum_download_shard": (C.c_int, [_vp, C.c_size_t, _u64p, _f64p, C.c_size_t,
                                               C.POINTER(C.c_size_t)]),
    "iqcc_gpu_psum_gather": (C.c_int, [_vp, _u64p, _f64p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "iqcc_gpu_psum_dress": (C.c_int, [_vp, _u64p, C.c_double, C.c_double, C.c_double, C.c_size_t, _vp,
                                      C.c_size_t, C.POINTER(C.c_size_t), C.POINTER(CompressStatsC),
                                      C.POINTER(C.c_size_t)]),
    "iqcc_gpu_psum_expect": (C.c_int, [_vp, _f64p, C.POINTER(C.c_double)]),
    "iqcc_gpu_psum_qmf_energy_gradient": (C.c_int, [_vp, _f64p, _f64p, C.POINTER(C.c_double), _f64p]),
    "iqcc_gpu_psum_gradients": (C.c_int, [_vp, _f64p, _u64p, C.c_size_t, C.c_int, _f64p]),
    "iqcc_gpu_psum_rebalance": (C.c_int, [_vp, C.c_double, _szp]),
}

EXPORTED = tuple(_SIGS)


def _load() -> C.CDLL:
    try:
        build()
    except Exception as e:  # pragma: no cover - surfaced as ImportError
        raise ImportError(f"cannot build the B200 engine ({LIB_PATH}): {e}") from e
    try:
        lib = C.CDLL(LIB_PATH)
    except OSError as e:
        raise ImportError(f"cannot load the B200 engine {LIB_PATH}: {e}") from e
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def check(status: int) -> None:
    """Map a C-ABI status onto the reference's exception types."""
    if status == IQCC_OK:
        return
    msg = lib.iqcc_gpu_last_error().decode(errors="replace")
    if status == IQCC_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if status == IQCC_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)  # std::runtime_error / CUDA failure


_initialised_device = None


def init(device: int | None = None) -> None:
    """Bind the engine to a device (once per process).  With no argument an
    already initialised engine is kept; otherwise torch's current device."""
    global _initialised_device
    if device is None:
        if _initialised_device is not None:
            return
        try:
            import torch
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        except Exception:
            device = 0
    if _initialised_device == device:
        return
    check(lib.iqcc_gpu_init(device))
    _initialised_device = device


def init_thread(device: int) -> None:
    """Give the calling host thread its own engine context on `device` (its
    own stream, scratch, block cache and page-locked staging; the C-ABI's
    contexts are per host thread).  Calls from different threads then run
    concurrently on the device: one call's uploads overlap another's
    dressing and downloads.  Pair with finalize_thread()."""
    check(lib.iqcc_gpu_init(device))


def finalize_thread() -> None:
    """Release the calling thread's engine context (device memory, caches)."""
    check(lib.iqcc_gpu_finalize())


def launch_count() -> int:
    return int(lib.iqcc_gpu_launch_count())


def profile(enable: bool) -> None:
    check(lib.iqcc_gpu_profile_enable(int(enable)))


def profile_get(name: str):
    ms, n = C.c_double(0), C.c_uint64(0)
    check(lib.iqcc_gpu_profile_get(name.encode(), C.byref(ms), C.byref(n)))
    return ms.value, n.value


def profile_bytes(name: str) -> float:
    b = C.c_double(0)
    check(lib.iqcc_gpu_profile_bytes(name.encode(), C.byref(b)))
    return b.value


def profile_reset() -> None:
    check(lib.iqcc_gpu_profile_reset())


def set_stream(handle: int | None) -> None:
    check(lib.iqcc_gpu_set_stream(handle))
