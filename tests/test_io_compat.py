"""Byte compatibility of the drop-in's file outputs with the reference's own
writers and readers:

* SWIH1 table dumps (integral_tables.cpp:167-206): the GPU build's save_file
  is byte-identical to the reference's for the same image; a reference-
  written dump loads here and re-saves byte-identically; a dump written here
  loads in the reference with the oracle's tables.
* likelihood-map CSV (%.9g) and PGM (map_to_gray) outputs
  (matching.cpp:225-252, the CLI pipeline's byte-identity check,
  cli_pipeline.sh:22-31), and the PGM round trip.
* the bench CSV schema (bench.cpp:132-143).
The C++ side runs tests/cpp/io_tool.cpp over libswih_b200.so; the reference
side is oracle/_ref/libswihref.so."""
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "tests", "cpp", "build", "io_tool")


def tool(*args):
    if not os.path.exists(TOOL):
        from paper_1705_03524_b200 import build
        build.build_cpp_tests()
    r = subprocess.run([TOOL, *map(str, args)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    return r


def write_pgm(path, img):
    h, w = img.shape
    with open(path, "wb") as f:
        f.write(f"P5\n{w} {h}\n255\n".encode() + img.tobytes())


@pytest.mark.parametrize("w,h,bins", [(3, 3, 2), (57, 41, 8), (300, 200, 16)])
def test_swih1_dumps_byte_identical(tmp_path, ref, oracle, w, h, bins):
    img = oracle.random_gray(w, h, 1000 + w)
    fi = oracle.quantize_gray8(img, bins)
    fi.tofile(tmp_path / "fi.u16")
    ours, theirs = tmp_path / "ours.swih", tmp_path / "ref.swih"
    tool("dump", tmp_path / "fi.u16", w, h, bins, ours)
    rt = ref.tables(fi, bins)
    rt.save(str(theirs))
    assert ours.read_bytes() == theirs.read_bytes()
    # a reference-written dump loads here and re-saves byte-identically
    again = tmp_path / "again.swih"
    tool("resave", theirs, again)
    assert again.read_bytes() == theirs.read_bytes()
    # our dump loads in the reference, with the oracle's tables
    lw, lh, lb, p, x, y = ref.load_tables(str(ours))
    assert (lw, lh, lb) == (w, h, bins)
    op, ox, oy = oracle.build_tables(fi, bins)
    assert (p == op).all() and (x == ox).all() and (y == oy).all()


def test_swih1_load_errors(tmp_path):
    bad = tmp_path / "bad.swih"
    bad.write_bytes(b"SWIH0" + bytes(20))
    r = subprocess.run([TOOL, "resave", bad, tmp_path / "x.swih"], capture_output=True,
                       text=True)
    assert r.returncode == 1 and "io_tool:" in r.stderr


@pytest.mark.parametrize("kind,method,rings", [(O.MANHATTAN, O.SWIH, 1),
                                               (O.GAUSS_CHEB, O.CAKE, 6),
                                               (O.UNIFORM, O.PLAIN, 1)])
def test_map_csv_and_pgm_byte_identical(tmp_path, ref, oracle, kind, method, rings):
    img = oracle.random_gray(96, 80, 31)
    img = np.ascontiguousarray(((img.astype(np.uint16) + np.roll(img, 1, 1)) // 2)
                               .astype(np.uint8))
    write_pgm(tmp_path / "search.pgm", img)
    kw = kh = 11
    tx, ty = 40, 35
    bins = 16
    tool("map", tmp_path / "search.pgm", bins, kind, kw, kh, method, rings, tx, ty,
         tmp_path / "ours.csv", tmp_path / "ours.pgm")
    k = O.kernel(kind, kw, kh, 0.5)
    templ = np.ascontiguousarray(img[ty - 5:ty + 6, tx - 5:tx + 6])
    model = ref.target_model(templ, bins, k, method, rings)
    scores, _ = ref.likelihood_map(img, bins, model, k, method, 0, rings, 0,
                                   want_scores=True)
    ref.write_map_files(scores, 5, 5, str(tmp_path / "ref.csv"), str(tmp_path / "ref.pgm"))
    assert (tmp_path / "ours.csv").read_bytes() == (tmp_path / "ref.csv").read_bytes()
    assert (tmp_path / "ours.pgm").read_bytes() == (tmp_path / "ref.pgm").read_bytes()


def test_pgm_round_trip(tmp_path, oracle):
    img = oracle.random_gray(37, 23, 21)
    src = tmp_path / "in.pgm"
    with open(src, "wb") as f:  # header with a comment line, as the reference reader skips
        f.write(b"P5\n# comment\n37 23\n255\n" + img.tobytes())
    tool("pgm", src, tmp_path / "out.pgm")
    out = (tmp_path / "out.pgm").read_bytes()
    assert out == b"P5\n37 23\n255\n" + img.tobytes()


@pytest.mark.parametrize("method", [O.SWIH, O.BRUTE, O.CAKE, O.PLAIN])
def test_bench_csv_schema(tmp_path, ref, method):
    out = tmp_path / "ours.csv"
    tool("bench", 48, 40, 8, 5, method, out)
    lines = out.read_text().splitlines()
    assert lines[0] == "method,width,height,kw,kh,bins,build_ms,query_total_ms,query_mean_us"
    f = lines[1].split(",")
    assert f[0] == ["swih", "brute", "cake", "plain"][method]
    rec = dict(method=f[0], width=int(f[1]), height=int(f[2]), kw=int(f[3]), kh=int(f[4]),
               bins=int(f[5]), build_ms=float(f[6]), query_total_ms=float(f[7]),
               query_mean_us=float(f[8]))
    assert (rec["width"], rec["height"], rec["kw"], rec["bins"]) == (48, 40, 5, 8)
    assert rec["query_mean_us"] == pytest.approx(rec["query_total_ms"] * 1000 / (44 * 36),
                                                 rel=1e-3, abs=1e-4)
    if method == O.BRUTE:
        assert rec["build_ms"] == 0.0
    ref.write_bench_csv(rec, str(tmp_path / "ref.csv"))
    assert out.read_bytes() == (tmp_path / "ref.csv").read_bytes()
