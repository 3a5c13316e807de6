"""The C-ABI library loads and exports every symbol include/mfb.h declares.

No device calls here (CPU-only CI): dlopen + dlsym, plus a check that the
product raises instead of falling back to CPU when no device is present.
"""

import ctypes
import os
import re

import pytest

from conftest import ROOT, has_gpu


def _declared():
    text = open(os.path.join(ROOT, "include", "mfb.h")).read()
    return sorted(set(re.findall(r"\b(mfb_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_and_exports_header_symbols():
    from paper_1802_06263_b200 import _build, _lib
    so = _build.build()
    lib = ctypes.CDLL(so)
    declared = _declared()
    assert declared, "no symbols parsed from mfb.h"
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_lib.exported_symbols()) == declared
    loaded = _lib.load()
    assert loaded.mfb_version().decode().startswith("mfb-b200")
    # provenance: the library carries the hash of the sources it was built from
    from paper_1802_06263_b200 import _build
    assert loaded.mfb_version().decode().endswith("src " + _build.source_hash())


def test_sass_has_fp64_tensor_instructions():
    import shutil
    import subprocess
    from paper_1802_06263_b200 import _build
    so = _build.build()
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", so], capture_output=True, text=True).stdout
    assert "DMMA" in sass
    assert "sm_100a" in subprocess.run([tool, "-lelf", so], capture_output=True,
                                       text=True).stdout or "sm_100" in sass


@pytest.mark.skipif(has_gpu(), reason="checks the no-device path")
def test_no_cpu_fallback_without_device():
    from conftest import case_from_golden
    from paper_1802_06263_b200.errors import NativeLibraryError
    from paper_1802_06263_b200.interface import run_method
    _, problem, grid, _ = case_from_golden("cfg1")
    with pytest.raises(NativeLibraryError):
        run_method(problem, grid, method="S3", tol=1e-11)


def test_method_and_cap_errors_before_device_work():
    from conftest import case_from_golden
    from paper_1802_06263_b200.errors import SizeCapError
    from paper_1802_06263_b200.interface import _check_basis_cap, run_method
    _, problem, grid, _ = case_from_golden("cfg1")
    with pytest.raises(ValueError, match="unknown method"):
        run_method(problem, grid, method="S9")
    with pytest.raises(SizeCapError, match="basis"):
        _check_basis_cap([8 * 12 * 12], 1e-9)
