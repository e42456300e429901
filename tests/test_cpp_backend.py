# SPDX-License-Identifier: Apache-2.0
"""The reference-side C++ binding (cpp_api/: hmi::sched::CudaBackend, compiled against the
reference's unchanged public headers) driven by a C++ caller holding the reference's own
types; see tests/cpp/test_cuda_backend.cpp. The program is built in the build container
(`make cppapi`, which needs /root/reference for the headers and the reference library) and
travels to the GPU box as a binary."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "cpp_api", "_build", "test_cuda_backend")


def _binary():
    if not os.path.exists(BIN) and os.path.isdir("/root/reference/proj/include"):
        subprocess.run(["make", "-C", ROOT, "cppapi"], check=True, capture_output=True)
    if not os.path.exists(BIN):
        pytest.skip("cpp_api/_build/test_cuda_backend not built (make cppapi needs the reference headers)")
    return BIN


def test_status_codes_map_to_reference_exceptions():
    """Every ABI status code rethrows as the reference's exception class (errors.hpp:10-68),
    FormatError with its byte offset; no GPU needed."""
    out = subprocess.run([_binary(), "--status-only"], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stderr
    assert json.loads(out.stdout.strip().splitlines()[-1])["status_mapping"] is True


@pytest.mark.gpu
def test_cpp_backend_matches_reference_path(tmp_path):
    """HeadOutput from CudaBackend::infer / run for InferBatches over artefacts built by the
    reference's own generators and builders equals higher_stack_forward(retrieve_sequence(...))
    within the tolerance (labels exactly); run() equals infer() bit for bit; replace / erase /
    re-register; every error class the backend can raise through the ABI."""
    out = subprocess.run([_binary(), str(tmp_path)], capture_output=True, text=True, timeout=900)
    print(out.stdout, out.stderr[-4000:])
    assert out.returncode == 0, out.stderr[-4000:]
    rec = json.loads(out.stdout.strip().splitlines()[-1])
    assert rec["failures"] == 0
    assert rec["max_rel_err"] <= 2e-2
    assert rec["label_agree"] == rec["labels"] > 0
    assert rec["run_equals_infer"] is True
