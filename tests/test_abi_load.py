"""CPU: libswg.so builds for sm_100a, loads, and exports every entry point
include/swg.h declares.  No compute calls (there is no GPU here); without a
device the library must fail loudly, never fall back."""
import ctypes
import os
import subprocess

import pytest

from paper_1705_03524_b200 import build, swg


def test_library_builds_and_loads():
    path = build.build()
    assert os.path.exists(path)
    assert swg.lib().swg_abi_version() == 1


def test_every_declared_symbol_is_exported():
    declared = swg.exported_symbols()
    assert len(declared) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", build.LIB], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines()}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing


def test_cubin_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(swg.NoDeviceError):
        swg.Context(0)


def test_status_codes_map_to_reference_classes():
    assert swg._BY_CODE[8] is swg.CapacityError
    assert swg._BY_CODE[7] is swg.WindowOutOfBoundsError
    assert swg._BY_CODE[6] is swg.UnsupportedKernelError
    assert issubclass(swg.SizeError, swg.Error)
