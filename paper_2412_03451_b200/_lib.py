"""ctypes binding of the C ABI declared in include/psplat_b200.h.

The shared library is built in-tree (``paper_2412_03451_b200/lib/libpsplat_b200.so``,
sm_100a) by ``__graft_entry__.build()`` / ``make -C paper_2412_03451_b200/csrc``.
There is no fallback: importing works without a GPU (so the CPU test suite can
check the exported symbols), but every compute entry point fails loudly with
``PsgCudaError`` when no B200 is present, and loading fails with ImportError when
the library was not built.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PSG_LIB", os.path.join(HERE, "lib", "libpsplat_b200.so"))

PSG_OK, PSG_EINVAL, PSG_ECUDA, PSG_ENONFINITE, PSG_ENCCL, PSG_ENOMEM, PSG_EIO = range(7)
PSG_FP32, PSG_FP64, PSG_MIXED = 0, 1, 2
PSG_STEP_WRITE_MAPS, PSG_STEP_NO_BACKWARD = 1, 2
PSG_NCCL_ID_BYTES = 128
PSG_ABI_VERSION = 4  # include/psplat_b200.h; a stale library is refused at load


class PsgError(RuntimeError):
    pass


class PsgCudaError(PsgError):
    pass


class PsgNcclError(PsgError):
    pass


class psg_render_config(C.Structure):
    _fields_ = [
        ("max_records", C.c_int32), ("normalize_by_alpha", C.c_int32),
        ("tile_size", C.c_int32), ("threads", C.c_int32),
        ("weight_floor", C.c_double), ("t_near", C.c_double), ("parallel_eps", C.c_double),
        ("alpha_floor", C.c_double), ("alpha1", C.c_double), ("alpha2", C.c_double),
    ]


class psg_camera(C.Structure):
    _fields_ = [
        ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
        ("width", C.c_int32), ("height", C.c_int32),
        ("rot_wc", C.c_double * 9), ("t_wc", C.c_double * 3),
    ]


class psg_stats(C.Structure):
    _fields_ = [
        ("views", C.c_int64), ("pixels", C.c_int64), ("tiles", C.c_int64),
        ("pairs", C.c_int64), ("big_tiles", C.c_int64), ("zbound_violations", C.c_int64),
        ("pixel_pairs", C.c_int64), ("live_records", C.c_int64),
        ("cull_checks", C.c_int64), ("cull_misses", C.c_int64), ("replays", C.c_int64),
    ]


class psg_optim_config(C.Structure):
    _fields_ = [
        ("lr_center", C.c_double), ("lr_radii", C.c_double), ("lr_rotation", C.c_double),
        ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
        ("split_interval", C.c_int64), ("split_grad_threshold", C.c_double),
        ("enable_split", C.c_int32), ("single_radii", C.c_int32),
        ("views_per_step", C.c_int32), ("check_ranks", C.c_int32),
        ("seed", C.c_uint64), ("radii_floor", C.c_double),
        ("lambda_base", C.c_double), ("lambda_rate", C.c_double), ("lambda_max", C.c_double),
    ]


_vp = C.c_void_p
_i32, _i64, _d = C.c_int32, C.c_int64, C.c_double
_ctx = C.c_void_p

# name -> (restype, argtypes); the header is the source of truth and
# tests/test_abi.py checks that this table and the exports cover it.
SIGNATURES = {
    "psg_last_error": (C.c_char_p, []),
    "psg_abi_version": (C.c_int, []),
    "psg_default_config": (None, [C.POINTER(psg_render_config)]),
    "psg_lambda_schedule": (_d, [_i64, _d, _d, _d]),
    "psg_create": (C.c_int, [C.c_int, C.c_int, C.POINTER(_ctx)]),
    "psg_destroy": (C.c_int, [_ctx]),
    "psg_set_stream": (C.c_int, [_ctx, _vp]),
    "psg_get_stream": (_vp, [_ctx]),
    "psg_set_config": (C.c_int, [_ctx, C.POINTER(psg_render_config)]),
    "psg_synchronize": (C.c_int, [_ctx]),
    "psg_set_planes": (C.c_int, [_ctx, _i64, _vp, _vp, _vp, _vp]),
    "psg_num_planes": (_i64, [_ctx]),
    "psg_render_view": (C.c_int, [_ctx, C.POINTER(psg_camera), _d, C.c_int, _vp, _vp, _vp, _vp, _vp]),
    "psg_render_loss": (C.c_int, [_ctx, C.POINTER(psg_camera), _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                  _vp, _vp]),
    "psg_backward": (C.c_int, [_ctx, C.POINTER(psg_camera), _d, C.c_int, _vp, _vp, _vp, _vp, _vp,
                               _vp, C.POINTER(_i64)]),
    "psg_set_views": (C.c_int, [_ctx, C.c_int, _vp, _vp, _vp]),
    "psg_update_targets": (C.c_int, [_ctx, C.c_int, C.c_int, _vp, _vp]),
    "psg_get_targets": (C.c_int, [_ctx, C.c_int, _vp, _vp]),
    "psg_render_ground_truth": (C.c_int, [_ctx, C.c_int, _vp]),
    "psg_step": (C.c_int, [_ctx, _vp, C.c_int, _d, _d, C.c_int]),
    "psg_step_host": (C.c_int, [_ctx, C.c_int, C.c_int, _d, _d, C.c_int, _vp, _vp, C.c_int]),
    "psg_zero_grads": (C.c_int, [_ctx]),
    "psg_set_deterministic": (C.c_int, [_ctx, C.c_int]),
    "psg_finalize_grads": (C.c_int, [_ctx, C.POINTER(_i64)]),
    "psg_read_grads": (C.c_int, [_ctx, _vp, C.POINTER(_d)]),
    "psg_read_view_losses": (C.c_int, [_ctx, _vp, C.c_int]),
    "psg_read_step_maps": (C.c_int, [_ctx, C.c_int, _vp, _vp, _vp]),
    "psg_get_stats": (C.c_int, [_ctx, C.POINTER(psg_stats)]),
    "psg_set_pair_limit": (C.c_int, [_ctx, _i64]),
    "psg_debug_probe": (C.c_int, [_ctx, _vp]),
    "psg_reset_stats": (C.c_int, [_ctx]),
    "psg_set_timing": (C.c_int, [_ctx, C.c_int]),
    "psg_get_kernel_ms": (C.c_int, [_ctx, C.POINTER(_d), C.POINTER(C.c_int)]),
    "psg_debug_bins": (_i64, [_ctx, C.POINTER(psg_camera), _d, _vp, _vp, _i64]),
    "psg_nccl_unique_id": (C.c_int, [_vp]),
    "psg_comm_init": (C.c_int, [_ctx, _vp, C.c_int, C.c_int]),
    "psg_allreduce_grads": (C.c_int, [_ctx]),
    "psg_comm_destroy": (C.c_int, [_ctx]),
    "psg_default_optim_config": (None, [C.POINTER(psg_optim_config)]),
    "psg_view_for_slot": (_i64, [C.c_uint64, _i64, _i64]),
    "psg_optim_reset": (C.c_int, [_ctx, _i64, _i64]),
    "psg_optim_step": (C.c_int, [_ctx, C.POINTER(psg_optim_config), C.POINTER(_d)]),
    "psg_optim_apply": (C.c_int, [_ctx, C.POINTER(psg_optim_config)]),
    "psg_optim_step_local": (C.c_int, [_ctx, C.POINTER(psg_optim_config), C.c_int, C.c_int]),
    "psg_optim_step_finish": (C.c_int, [_ctx, C.POINTER(psg_optim_config), C.POINTER(_d)]),
    "psg_params_checksum": (C.c_int, [_ctx, C.POINTER(C.c_uint64)]),
    "psg_optim_maybe_split": (C.c_int, [_ctx, C.POINTER(psg_optim_config), C.POINTER(_i64)]),
    "psg_optim_run": (C.c_int, [_ctx, C.POINTER(psg_optim_config), _i64, _vp, _vp, _vp, _i64,
                                C.POINTER(_i64)]),
    "psg_set_grads": (C.c_int, [_ctx, _vp, _d]),
    "psg_get_planes": (C.c_int, [_ctx, _vp, _vp, _vp, _vp]),
    "psg_optim_get_state": (C.c_int, [_ctx, _vp, _vp, _vp, _vp, _vp, C.POINTER(_i64),
                                      C.POINTER(_i64)]),
    "psg_optim_set_state": (C.c_int, [_ctx, _vp, _vp, _vp, _vp, _vp, _i64, _i64]),
    "psg_merge_planes": (C.c_int, [_ctx, _vp, _d, _d, _d, C.c_int, _vp, _vp, _vp, _vp,
                                   C.POINTER(_i64)]),
    "psg_dataset_open": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(_vp)]),
    "psg_dataset_close": (C.c_int, [_vp]),
    "psg_dataset_size": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(_i64)]),
    "psg_dataset_cameras": (C.c_int, [_vp, _vp, _vp]),
    "psg_dataset_read": (C.c_int, [_vp, C.c_int, C.c_int, _vp, _vp, C.c_int]),
    "psg_load_dataset": (C.c_int, [_ctx, _vp, C.c_int, C.c_int]),
    "psg_write_map_f32": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, _vp]),
    "psg_read_map_f32": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), _vp,
                                   _i64]),
    "psg_refresh_target_counts": (C.c_int, [_ctx]),
    "psg_init_from_depth": (C.c_int, [_ctx, C.c_int, C.c_uint64, _d, C.POINTER(_i64)]),
    "psg_host_alloc": (_vp, [C.c_size_t]),
    "psg_host_free": (None, [_vp]),
}

_LIB = None


def lib() -> C.CDLL:
    """Load the in-tree CUDA library (ImportError if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if L.psg_abi_version() != PSG_ABI_VERSION:
            raise ImportError(f"{LIB_PATH} has ABI {L.psg_abi_version()}, this binding expects "
                              f"{PSG_ABI_VERSION}: rebuild it (make -C paper_2412_03451_b200/csrc)")
        _LIB = L
    return _LIB


def last_error() -> str:
    msg = lib().psg_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> None:
    """Map a psg_status to the exception type the reference throws."""
    if status == PSG_OK:
        return
    msg = last_error() or what
    if status == PSG_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if status in (PSG_ENONFINITE, PSG_EIO):
        raise RuntimeError(msg)  # std::runtime_error
    if status == PSG_ECUDA:
        raise PsgCudaError(msg)
    if status == PSG_ENCCL:
        raise PsgNcclError(msg)
    raise PsgError(f"{what}: status {status}: {msg}")
