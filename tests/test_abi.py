"""CPU-side checks of the C-ABI boundary: the library loads and exports every
symbol include/fibar_b200.h declares (no compute calls without a GPU)."""

import os
import re
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def declared():
    src = open(os.path.join(ROOT, "include", "fibar_b200.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char \*)\s*(fibar_\w+)\s*\(", src, re.M)))


def test_header_declares_entry_points():
    names = declared()
    assert "fibar_create" in names and "fibar_process" in names and "fibar_render" in names
    assert len(names) >= 12


def test_library_exports_every_declared_symbol():
    from paper_2510_20071_b200 import build as nb, _native
    nb.build()
    out = subprocess.run(["nm", "-D", "--defined-only", nb.OUT], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(fibar_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    lib = _native.load()
    for n in declared():
        getattr(lib, n)
    assert set(_native.EXPORTED) == set(declared())


def test_library_targets_sm100a_only():
    from paper_2510_20071_b200 import build as nb
    nb.build()
    out = subprocess.run(["cuobjdump", "--list-elf", nb.OUT], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cuda_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2510_20071_b200.core import SensorGeometry, compute_params
    from paper_2510_20071_b200.errors import DeviceError
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    g = SensorGeometry(8, 8)
    with pytest.raises(DeviceError):
        ReconstructionEngine(g, compute_params(40.0, geometry=g))
