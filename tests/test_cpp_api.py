"""The reference's C++ operator API as a drop-in (include/widthfold/*.hpp at the
reference's include paths, libwidthfold.so): tests/cpp/test_reference_api.cpp
is a reference-style C++ caller built against only those headers.

CPU: the binary links and its host-only criteria pass (DenseTensor values,
the error taxonomy, legality, MAC accounting). GPU: every criterion, incl. the
Appendix-A vectors the reference's own module produced (tests/golden/appendix_a.npz,
dumped here as raw float32 files) compared bitwise.
"""
import os
import subprocess

import numpy as np
import pytest

from tests.conftest import GOLDEN, ROOT

BIN = os.path.join(ROOT, "tests", "cpp", "test_reference_api")


def _run(*args):
    if not os.path.exists(BIN):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2601_11608_b200", "csrc"), "-j4"], check=True,
                       capture_output=True)
    return subprocess.run([BIN, *args], capture_output=True, text=True, timeout=600)


def test_header_only_caller_links_and_host_criteria_pass():
    r = _run("--host-only")
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("[PASS]") == 2


@pytest.mark.gpu
def test_reference_caller_runs_on_device(tmp_path):
    with np.load(os.path.join(GOLDEN, "appendix_a.npz")) as z:
        for k in z.files:
            a = np.ascontiguousarray(z[k], dtype=np.float32)
            a.tofile(tmp_path / f"{k}.f32")
            (tmp_path / f"{k}.shape").write_text(" ".join(str(e) for e in a.shape))
    r = _run(str(tmp_path))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[FAIL]" not in r.stdout and r.stdout.count("[PASS]") == 8, r.stdout
    assert "skipped" not in r.stdout
