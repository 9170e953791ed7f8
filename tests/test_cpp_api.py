"""The reference-compatible C++ API (include/swih/*.hpp) over libswg.

CPU: the library and the C++ test binary build, and the API symbols are
exported.  GPU: the C++ suite (tests/cpp/test_api.cpp, the reference suites'
properties and known answers restated) passes against the B200 path."""
import subprocess

import pytest

from paper_1705_03524_b200 import build


def test_cpp_layer_builds_and_exports_the_api():
    lib = build.build_cpp()
    syms = subprocess.run(["nm", "-DC", "--defined-only", lib], capture_output=True, text=True,
                          check=True).stdout
    for name in ["swih::IntegralTableSet::build", "swih::likelihood_map", "swih::peak",
                 "swih::swih_query_into", "swih::decompose", "swih::WeddingCakePlan::histogram_into",
                 "swih::BruteForcePlan::counts_into", "swih::quantize_image", "swih::target_model",
                 "swih::IntegralTableSet::save", "swih::IntegralTableSet::load"]:
        assert name in syms, name
    ldd = subprocess.run(["ldd", lib], capture_output=True, text=True).stdout
    assert "libswg.so" in ldd
    assert build.build_cpp_tests()


@pytest.mark.gpu
def test_cpp_api_suite_on_gpu():
    exe = build.build_cpp_tests()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failed cases" in r.stdout
