# SPDX-License-Identifier: Apache-2.0
"""ctypes binding of the in-tree C-ABI library ``_lib/libhmi_b200.so``.

The product path has no CPU fallback: if the shared library is missing this
module raises on first use (:func:`lib`). Status codes become the Python
mirrors of the reference's exception classes (proj/include/hmi/errors.hpp).
"""
from __future__ import annotations

import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HMI_LIB_PATH") or os.path.join(_HERE, "_lib", "libhmi_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "hmi_gpu.h")

_lib = None


class HmiError(RuntimeError):
    code = -1


class DimensionError(HmiError, ValueError):
    code = 1


class VocabularyError(HmiError, IndexError):
    code = 2


class ConflictError(HmiError):
    code = 3


class CapacityError(HmiError):
    code = 4


class RoutingError(HmiError):
    code = 5


class ConfigError(HmiError):
    code = 6


class BuildError(HmiError):
    code = 7


class SchedulingBugError(HmiError):
    code = 8


class FormatError(HmiError):
    code = 9


class CudaError(HmiError):
    code = 100


ERRORS = {c.code: c for c in (DimensionError, VocabularyError, ConflictError, CapacityError,
                              RoutingError, ConfigError, BuildError, SchedulingBugError,
                              FormatError, CudaError)}
STATUS_NAMES = {0: "OK", **{k: v.__name__ for k, v in ERRORS.items()}}


class ModelConfig(ctypes.Structure):
    """hmi_model_config == ModelConfig (proj/include/hmi/transformer/config.hpp:10-24)."""

    _fields_ = [(n, ctypes.c_uint32) for n in (
        "hidden_size", "heads", "lower_layers", "higher_layers", "ffn_size", "vocab_size",
        "mode", "max_fragment", "seed")]


class Options(ctypes.Structure):
    _fields_ = [("precision", ctypes.c_uint32), ("max_batch", ctypes.c_uint32),
                ("max_seq", ctypes.c_uint32), ("bottleneck", ctypes.c_uint32),
                ("max_labels", ctypes.c_uint32), ("pipeline_mode", ctypes.c_uint32),
                ("pool_bytes", ctypes.c_uint64), ("max_tasks", ctypes.c_uint32),
                ("max_instances", ctypes.c_uint32), ("max_heads", ctypes.c_uint32),
                ("max_versions", ctypes.c_uint32), ("max_new_tokens", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32)]


class LoadRecord(ctypes.Structure):
    _fields_ = [("task", ctypes.c_uint32), ("layer", ctypes.c_int32), ("hit", ctypes.c_int32),
                ("n_evicted", ctypes.c_uint32), ("bytes", ctypes.c_uint64),
                ("evicted_offset", ctypes.c_uint32), ("pad", ctypes.c_uint32)]


class TaskExport(ctypes.Structure):
    """hmi_task_export: where an exported task's HBM slots live (include/hmi_gpu.h)."""

    _fields_ = [("device", ctypes.c_int32), ("pid", ctypes.c_int32), ("arena", ctypes.c_uint64),
                ("ipc_handle", ctypes.c_uint8 * 64), ("slot_bytes", ctypes.c_uint64),
                ("fingerprint", ctypes.c_uint64), ("layers", ctypes.c_uint32),
                ("task_idx", ctypes.c_uint32), ("slot", ctypes.c_int32 * 64)]


class StageRecord(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_uint64), ("stage", ctypes.c_uint32), ("layer", ctypes.c_int32),
                ("worker", ctypes.c_uint32), ("pad", ctypes.c_uint32), ("start_ms", ctypes.c_double),
                ("end_ms", ctypes.c_double)]


def declared_symbols(header: str = HEADER_PATH) -> list[str]:
    """Every ``hmi_*`` function declared in the C header."""
    text = open(header).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hmi_[a-z0-9_]+)\s*\(", text)))


def _sig(L):
    vp, u32, i32, u64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int32, ctypes.c_uint64
    P = ctypes.POINTER
    f32p, f64p = P(ctypes.c_float), P(ctypes.c_double)
    u32p, i32p, u64p = P(u32), P(i32), P(u64)
    L.hmi_gpu_last_error.restype = ctypes.c_char_p
    L.hmi_gpu_create.argtypes = [ctypes.c_int, P(ModelConfig), P(Options), f32p, P(vp)]
    L.hmi_gpu_destroy.argtypes = [vp]
    L.hmi_gpu_upload_table.argtypes = [vp, u32, u32, u32, u32p, u32p, f32p]
    L.hmi_gpu_register_task.argtypes = [vp, u32, f32p]
    L.hmi_gpu_replace_task.argtypes = [vp, u32, f32p]
    L.hmi_gpu_unregister_task.argtypes = [vp, u32]
    L.hmi_gpu_register_head.argtypes = [vp, u32, u32, u32, f32p, f32p]
    L.hmi_gpu_bind_instance.argtypes = [vp, u32, u32, u32, u32]
    L.hmi_gpu_unbind_instance.argtypes = [vp, u32]
    L.hmi_gpu_infer_batch.argtypes = [vp, u32, u32p, u32p, u32, u32p, f32p, i32p, i32p,
                                      P(LoadRecord), u32, u32p, u32, u32p]
    L.hmi_gpu_infer_batch_device.argtypes = [vp, u32, u32p, vp, u32, vp, u32, vp, vp]
    L.hmi_gpu_generate.argtypes = [vp, u32, u32p, u32p, u32, u32p, u32, i32p, f32p]
    L.hmi_plot_builder_create.argtypes = [ctypes.c_int, P(ModelConfig), f32p, f32p, f32p, u32, u32,
                                          P(vp)]
    L.hmi_plot_builder_destroy.argtypes = [vp]
    L.hmi_plot_builder_stats.argtypes = [vp, f64p, u64p]
    L.hmi_plot_forward.argtypes = [vp, u32, u32p, u32p, f32p]
    L.hmi_plot_build_root.argtypes = [vp, u32, u32p, u32p, P(vp)]
    L.hmi_plot_derive_branch.argtypes = [vp, vp, u32, u32p, u32p, ctypes.c_double, P(vp)]
    L.hmi_plot_select_root.argtypes = [u32, u32, u32, u32p, u32p, P(vp)]
    L.hmi_plot_select_branch.argtypes = [u32, u32, u32p, u32p, ctypes.c_double, P(vp)]
    cp = ctypes.c_char_p
    L.hmi_plot_table_shape.argtypes = [vp, u32p, u32p]
    L.hmi_plot_table_load.argtypes = [cp, P(vp), u32p, u32p, u32p]
    L.hmi_plot_table_save.argtypes = [vp, cp, u32, u32, cp, u32]
    L.hmi_adapter_set_load.argtypes = [cp, ctypes.c_char_p, u32, u32p, u32p, u32p, f32p]
    L.hmi_model_load.argtypes = [cp, P(ModelConfig), f32p, f32p, f32p, f32p]
    L.hmi_gpu_upload_plot_table.argtypes = [vp, u32, u32, vp]
    L.hmi_gpu_register_task_file.argtypes = [vp, u32, cp]
    L.hmi_gpu_check_adapter_dims.argtypes = [vp, u32, u32, u32]
    L.hmi_gpu_register_tasks.argtypes = [vp, u32, u32p, P(f32p), u32]
    L.hmi_gpu_register_task_files.argtypes = [vp, u32, u32p, P(cp), u32]
    L.hmi_gpu_upload_plt1.argtypes = [vp, cp, u32p, u32p]
    L.hmi_gpu_export_task.argtypes = [vp, u32, P(TaskExport)]
    L.hmi_gpu_import_task.argtypes = [vp, u32, P(TaskExport), f32p, u64p]
    L.hmi_gpu_release_export.argtypes = [vp, u32, ctypes.c_int]
    L.hmi_plot_table_create.argtypes = [u32, u32, u32, u32p, u32p, u64p, f32p, P(vp)]
    L.hmi_plot_table_info.argtypes = [vp, u32p, u64p, u32p]
    L.hmi_plot_table_read.argtypes = [vp, u32p, u32p, u64p, f32p]
    L.hmi_plot_table_free.argtypes = [vp]
    L.hmi_gpu_trace.argtypes = [vp, ctypes.c_int]
    L.hmi_gpu_stage_trace.argtypes = [vp, ctypes.c_void_p, u32, u32p]
    L.hmi_gpu_copy_probe.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_size_t, ctypes.c_int,
                                     ctypes.c_int, f64p]
    L.hmi_gpu_submit_batch.argtypes = [vp, u32, u32p, u32p, u32, u32p, u64p]
    L.hmi_gpu_wait_batch.argtypes = [vp, u64, f32p, i32p]
    L.hmi_gpu_synchronize.argtypes = [vp]
    L.hmi_gpu_stream.argtypes = [vp]
    L.hmi_gpu_stream.restype = vp
    L.hmi_gpu_debug_routing.argtypes = [vp, i32p, i32p, i32p, i32p]
    L.hmi_gpu_debug_gather.argtypes = [vp, i32p, i32p, u32p]
    L.hmi_gpu_set_debug.argtypes = [vp, u32]
    L.hmi_gpu_debug_h0.argtypes = [vp, f64p]
    L.hmi_gpu_debug_hidden.argtypes = [vp, f32p]
    L.hmi_gpu_pool_stats.argtypes = [vp, u64p]
    L.hmi_gpu_pool_slot.argtypes = [vp, u32, u32, i32p]
    L.hmi_gpu_profile.argtypes = [vp, ctypes.c_int]
    L.hmi_gpu_profile_read.argtypes = [vp, f64p, u64p]
    L.hmi_gpu_profile_name.argtypes = [ctypes.c_int]
    L.hmi_gpu_profile_name.restype = ctypes.c_char_p
    L.hmi_pool_create.argtypes = [u64, P(vp)]
    L.hmi_pool_destroy.argtypes = [vp]
    L.hmi_pool_register.argtypes = [vp, u32, u32, u64]
    L.hmi_pool_op.argtypes = [vp, ctypes.c_int, u32, u32p, u32, P(LoadRecord), u32, u32p, u32,
                              P(i32)]
    L.hmi_pool_stats.argtypes = [vp, u64p]
    L.hmi_pool_create_placed.argtypes = [u64, u32, u32, P(vp)]
    L.hmi_pool_slot.argtypes = [vp, u32, u32, P(ctypes.c_int32)]
    L.hmi_generate_model.argtypes = [P(ModelConfig), f32p, f32p, f32p, f32p]
    L.hmi_generate_adapter.argtypes = [P(ModelConfig), u32, u64, f32p]
    L.hmi_generate_head.argtypes = [u32, u32, u64, f32p, f32p]
    L.hmi_gpu_counters.argtypes = [vp, u64p]
    L.hmi_gpu_h2d_probe.argtypes = [vp, u64, u32, P(ctypes.c_double)]


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"B200 extension not built: {LIB_PATH} is missing (run __graft_entry__.build())"
            )
        L = ctypes.CDLL(LIB_PATH)
        _sig(L)
        _lib = L
    return _lib


def last_error() -> str:
    msg = lib().hmi_gpu_last_error()
    return msg.decode() if msg else ""


def check(status: int) -> None:
    if status != 0:
        cls = ERRORS.get(status, HmiError)
        raise cls(f"[{STATUS_NAMES.get(status, status)}] {last_error()}")
