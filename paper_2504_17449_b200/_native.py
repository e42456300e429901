# SPDX-License-Identifier: Apache-2.0
"""ctypes loader for the in-tree C-ABI library ``_lib/libhmi_b200.so``.

The product path has no CPU fallback: if the shared library is missing or does
not export the symbols declared in ``include/hmi_gpu.h`` this module raises at
import time of :func:`lib`.
"""
from __future__ import annotations

import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libhmi_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "hmi_gpu.h")

_lib = None

STATUS_NAMES = {
    0: "OK",
    1: "DimensionError",
    2: "VocabularyError",
    3: "ConflictError",
    4: "CapacityError",
    5: "RoutingError",
    6: "ConfigError",
    7: "BuildError",
    8: "SchedulingBugError",
    9: "FormatError",
    100: "CudaError",
}


def declared_symbols(header: str = HEADER_PATH) -> list[str]:
    """Every ``hmi_*`` function declared in the C header."""
    text = open(header).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hmi_[a-z0-9_]+)\s*\(", text)))


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"B200 extension not built: {LIB_PATH} is missing (run __graft_entry__.build())"
            )
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.hmi_gpu_last_error.restype = ctypes.c_char_p
    return _lib


def last_error() -> str:
    msg = lib().hmi_gpu_last_error()
    return msg.decode() if msg else ""
