# SPDX-License-Identifier: Apache-2.0
"""The C-ABI library loads and exports every symbol include/hmi_gpu.h declares
(no compute calls: runs without a GPU)."""
import ctypes

from paper_2504_17449_b200 import _native


def test_header_symbols_exported():
    lib = _native.lib()
    declared = _native.declared_symbols()
    assert len(declared) >= 30
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing


def test_status_codes_match_reference_error_classes():
    # errors.hpp:10-68 order; see include/hmi_gpu.h
    names = [_native.STATUS_NAMES[i] for i in range(1, 10)]
    assert names == ["DimensionError", "VocabularyError", "ConflictError", "CapacityError",
                     "RoutingError", "ConfigError", "BuildError", "SchedulingBugError",
                     "FormatError"]


def test_create_rejects_invalid_config_without_gpu():
    lib = _native.lib()
    cfg = _native.ModelConfig(100, 3, 1, 1, 64, 10, 0, 3, 7)  # 100 % 3 != 0
    opts = _native.Options(0, 8, 128, 8, 4, 2, 0, 4, 4, 4, 8)
    w = (ctypes.c_float * 1)()
    h = ctypes.c_void_p()
    rc = lib.hmi_gpu_create(0, ctypes.byref(cfg), ctypes.byref(opts), w, ctypes.byref(h))
    assert rc == 6 and "multiple of heads" in _native.last_error()
    cfg = _native.ModelConfig(256, 4, 1, 1, 1024, 10, 0, 4, 7)  # n = 4 not in {1,2,3,5}
    rc = lib.hmi_gpu_create(0, ctypes.byref(cfg), ctypes.byref(opts), w, ctypes.byref(h))
    assert rc == 6 and "max_fragment" in _native.last_error()
