"""The full-size oracle (oracle/swih_fastmap.c, bin-outer) against the
window-by-window restatement (orc_likelihood_map, pinned to the reference
in test_oracle_golden.py): bit-identical maps for every exact method,
kernel and similarity; exact peaks for the declared exponential kernel's
two-phase map.  CPU only."""
import numpy as np
import pytest

from oracle import oracle as O

orc = O.Oracle()


def _scene(w, h, bins, seed):
    rng = np.random.default_rng(seed)
    # smooth-ish field so bins form regions (sparse and dense bins both occur)
    img = rng.integers(0, 256, size=(h, w)).astype(np.float64)
    for _ in range(2):
        img = (img + np.roll(img, 1, 0) + np.roll(img, 1, 1) + np.roll(img, -1, 1)) / 4
    img = np.clip(img, 0, 255).astype(np.uint8)
    return orc.quantize_gray8(img, bins)


CASES = [
    (O.MANHATTAN, O.SWIH, 1), (O.UNIFORM, O.SWIH, 1), (O.UNIFORM, O.PLAIN, 1),
    (O.MANHATTAN, O.BRUTE, 1), (O.EUCLID_QUAD, O.BRUTE, 1),
    (O.GAUSS_CHEB, O.CAKE, None), (O.GAUSS_CHEB, O.CAKE, 3), (O.CHEBYSHEV, O.CAKE, None),
    (O.MANHATTAN, O.CAKE, 2),
]


@pytest.mark.parametrize("kind,method,rings", CASES)
@pytest.mark.parametrize("sim", [O.BHATTACHARYYA, O.INTERSECTION])
@pytest.mark.parametrize("kw,kh", [(9, 7), (13, 13), (1, 5)])
def test_fast_map_bit_identical(kind, method, rings, sim, kw, kh):
    bins = 8
    fi = _scene(47, 38, bins, 11 + kw + kind)
    k = O.kernel(kind, kw, kh, 0.5)
    r = rings if rings else min(kw, kh) // 2 + 1
    r = min(r, min(kw, kh) // 2 + 1)
    tm = O.SWIH if method == O.PLAIN else method
    model = orc.target_model(fi[3:3 + kh, 5:5 + kw].copy(), bins, k,
                             O.PLAIN if method == O.PLAIN else tm, r)
    want = orc.likelihood_map(fi, bins, model, k, method, sim, rings=r)
    got, pk, _ = orc.fast_map(fi, bins, model, k, method, sim, rings=r, threads=3)
    assert got.shape == want.shape
    assert (got.view(np.int64) == want.view(np.int64)).all()
    assert pk == orc.peak(want, (kw - 1) // 2, (kh - 1) // 2)


def test_fast_map_threads_and_sparse_bins():
    """Thread chunking and empty bins (skipped) change nothing."""
    bins = 32
    fi = _scene(61, 52, bins, 5)
    fi[fi == 7] = 6  # bin 7 empty
    k = O.kernel(O.MANHATTAN, 11, 11)
    model = orc.target_model(fi[10:21, 10:21].copy(), bins, k)
    a, pa, _ = orc.fast_map(fi, bins, model, k, threads=1)
    b, pb, _ = orc.fast_map(fi, bins, model, k, threads=7)
    want = orc.likelihood_map(fi, bins, model, k)
    assert (a == want).all() and (b == want).all() and pa == pb


@pytest.mark.parametrize("sim", [O.BHATTACHARYYA, O.INTERSECTION])
@pytest.mark.parametrize("kw,kh,d", [(9, 9, 0.9375), (15, 11, 0.8), (21, 21, 0.97)])
def test_fast_map_exponential_two_phase(sim, kw, kh, d):
    """Declared exponential kernel: the separable phase-1 map is within 1e-10
    of the brute force everywhere, the re-scored windows are exact, and the
    peak (index and score bits) equals the brute-force map's."""
    bins = 8
    fi = _scene(58, 49, bins, 3 + kw)
    k = O.kernel(O.EXP_L1, kw, kh, d)
    model = orc.target_model(fi[7:7 + kh, 9:9 + kw].copy(), bins, k, O.BRUTE)
    want = orc.likelihood_map(fi, bins, model, k, O.BRUTE, sim)
    got, pk, n = orc.fast_map(fi, bins, model, k, O.BRUTE, sim, threads=4)
    assert np.abs(got - want).max() <= 1e-10
    assert n >= 1
    assert pk == orc.peak(want, (kw - 1) // 2, (kh - 1) // 2)
    exact = np.abs(got - want) == 0
    assert exact.sum() >= n


def test_fast_map_errors():
    fi = _scene(20, 20, 4, 1)
    m = np.full(4, 0.25)
    with pytest.raises(O.OracleError) as e:
        orc.fast_map(fi, 4, m, O.kernel(O.GAUSS_CHEB, 5, 5), O.SWIH)
    assert e.value.code == 6  # UnsupportedKernelError
    with pytest.raises(O.OracleError) as e:
        orc.fast_map(fi, 4, m, O.kernel(O.MANHATTAN, 4, 5), O.SWIH)
    assert e.value.code == 4  # InvalidKernelError
    with pytest.raises(O.OracleError) as e:
        orc.fast_map(fi, 4, m, O.kernel(O.MANHATTAN, 21, 5), O.SWIH)
    assert e.value.code == 11  # SizeError


def test_numpy_prefix_tables_equal_oracle_build():
    """The numpy table form the full-size GPU table tests use
    (test_gpu_fullsize._prefix_u32) equals the oracle build (pinned to the
    reference's IntegralTableSet::build) for plain / xramp / yramp."""
    from test_gpu_fullsize import _prefix_u32
    fi = _scene(37, 29, 6, 2)
    p, x, y = orc.build_tables(fi, 6)
    for b in range(6):
        want = _prefix_u32(fi, b, planes=3)
        assert (want[0] == p[b]).all() and (want[1] == x[b]).all() and (want[2] == y[b]).all()
