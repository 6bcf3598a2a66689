"""C-ABI checks that need no GPU: the library builds for sm_100a, loads, exports
every entry point include/sro.h declares, and fails loudly (no CPU fallback)
when no CUDA device is present."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2103_05857_b200 import build
    build.build()
    from paper_2103_05857_b200 import sro
    return sro.load_library()


def declared_entry_points():
    src = open(os.path.join(ROOT, "include", "sro.h")).read()
    return sorted(set(re.findall(r"^(?:sro_status|void|const char\*)\s+(sro_[a-z_]+)\s*\(", src, re.M)))


def test_header_declares_the_boundary():
    names = declared_entry_points()
    for n in ("sro_create", "sro_solve", "sro_gap", "sro_objective", "sro_get_plan"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2103_05857_b200 import sro
    for name in declared_entry_points():
        assert hasattr(lib, name), name
    assert set(declared_entry_points()) == set(sro.EXPORTED_SYMBOLS)
    assert lib.sro_version().decode().startswith("sro-b200")


def test_library_is_sm100a(lib):
    import subprocess
    from paper_2103_05857_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_gpu(lib):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2103_05857_b200 import sro
    with pytest.raises(sro.SroError) as e:
        sro.Solver(np.full(4, 0.25), np.full(2, 0.5), 1.0, C=np.ones((4, 2)))
    assert e.value.status == 7


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2103_05857_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower().replace("oracle's", ""), f
