"""Generate tests/golden/*.npz from the REFERENCE library itself.

Run in the build container (needs /root/reference):  python tests/golden/make_golden.py

Every array here is produced by oracle/_ref/libswihref.so, i.e. the
unmodified reference sources (/root/reference/proj/src) compiled by
oracle/Makefile, called through oracle/ref_shim.cpp.  The known-answer cases
mirror the reference's own tests (file:line in each entry's "source").  The
GPU box has no /root/reference: the tests read only these fixtures there.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1705_03524_b200 import synth  # noqa: E402


def save(name, source, **arrays):
    meta = {k: v for k, v in arrays.items() if not isinstance(v, np.ndarray)}
    arrs = {k: v for k, v in arrays.items() if isinstance(v, np.ndarray)}
    np.savez_compressed(os.path.join(HERE, name + ".npz"), meta=json.dumps(
        {"source": source, **meta}), **arrs)
    print(name, {k: v.shape for k, v in arrs.items()})


def cross3():
    return np.array([[10, 200, 10], [200, 10, 200], [10, 200, 10]], np.uint8)


def main():
    R = O.Ref()
    K = O.kernel

    # 1. cross image KATs (test_integral_tables.cpp:53-93, test_engine.cpp:99-147,
    #    test_baselines.cpp:21-48,50-101, test_matching.cpp:25-81)
    img = cross3()
    fi = R.quantize(img, 2)
    t = R.tables(fi, 2)
    man3 = K(O.MANHATTAN, 3, 3)
    save("cross3", "test_integral_tables.cpp:53-93; test_engine.cpp:99-147; "
         "test_baselines.cpp:21-101; test_matching.cpp:25-81",
         image=img, bins=2, fi=fi, plain=t.export(0), xramp=t.export(1), yramp=t.export(2),
         swih_man3=t.swih_query(1, 1, man3), plain_3x3=t.plain_query(1, 1, 3, 3),
         quad_tl=t.quadrant_histogram((0, 0, 1, 1), 1, 1, 1),
         model_man3=R.target_model(img, 2, man3),
         model_uni3=R.target_model(img, 2, K(O.UNIFORM, 3, 3)),
         cake_cheb3_r2=t.cake_histogram(K(O.CHEBYSHEV, 3, 3), 2, O.RING_MEAN, 1, 1),
         cake_man3_r2=t.cake_histogram(man3, 2, O.RING_MEAN, 1, 1),
         cake_man3_level=t.cake_histogram(man3, 2, O.RING_LEVEL, 1, 1),
         bhatt_example=np.array([R.similarity(0, np.array([7 / 15, 8 / 15]), np.array([.5, .5]))]))

    # 2. seeded random tables (test_integral_tables.cpp:95-110: 32x32 seed 99, b=8)
    img = R.random_gray(32, 32, 99)
    fi = R.quantize(img, 8)
    t = R.tables(fi, 8)
    save("tables_32x32_s99_b8", "test_integral_tables.cpp:95-110", image=img, bins=8,
         plain=t.export(0), xramp=t.export(1), yramp=t.export(2))

    # 3. clipped queries at every centre (test_engine.cpp:177-196)
    img = R.random_gray(15, 11, 8)
    fi = R.quantize(img, 4)
    t = R.tables(fi, 4)
    k = K(O.MANHATTAN, 7, 5)
    cl = np.array([[t.swih_query(cx, cy, k, O.CLIPPED) for cx in range(15)] for cy in range(11)])
    save("clipped_15x11_s8_b4", "test_engine.cpp:177-196", image=img, bins=4, counts=cl,
         kw=7, kh=5)

    # 4. swih vs brute maps + peak (test_matching.cpp:115-141)
    img = R.random_gray(40, 33, 2024)
    k = K(O.MANHATTAN, 9, 7)
    templ = np.ascontiguousarray(img[9:16, 12:21])
    model = R.target_model(templ, 8, k)
    m_b, p_b = R.likelihood_map(img, 8, model, k, O.SWIH, O.BHATTACHARYYA)
    m_i, p_i = R.likelihood_map(img, 8, model, k, O.SWIH, O.INTERSECTION)
    m_br, p_br = R.likelihood_map(img, 8, model, k, O.BRUTE, O.BHATTACHARYYA)
    m_pl, p_pl = R.likelihood_map(img, 8, R.target_model(templ, 8, k, O.PLAIN), k, O.PLAIN)
    save("map_40x33_s2024_b8_man9x7", "test_matching.cpp:115-141", image=img, bins=8,
         kw=9, kh=7, model=model, map_bhatt=m_b, peak_bhatt=np.array(p_b), map_inter=m_i,
         peak_inter=np.array(p_i), map_brute=m_br, map_plain=m_pl, peak_plain=np.array(p_pl))

    # 5. tiled template (test_matching.cpp:83-113), all four methods
    tile = cross3()
    search = np.array([[tile[y % 3, x % 3] for x in range(9)] for y in range(6)], np.uint8)
    out = {}
    for name, meth in (("swih", O.SWIH), ("brute", O.BRUTE), ("cake", O.CAKE), ("plain", O.PLAIN)):
        mdl = R.target_model(tile, 2, man3, meth, rings=2)
        out["model_" + name] = mdl
        out["map_" + name] = R.likelihood_map(search, 2, mdl, man3, meth, rings=2)[0]
    save("tiled_9x6", "test_matching.cpp:83-113", image=search, bins=2, **out)

    # 6. Gaussian-Chebyshev: cake (full rings, exact telescoping) and brute maps
    img = R.random_gray(48, 40, 60)
    kg = K(O.GAUSS_CHEB, 9, 9, 0.6)
    templ = np.ascontiguousarray(img[10:19, 20:29])
    mc = R.target_model(templ, 8, kg, O.CAKE, rings=5)
    mb = R.target_model(templ, 8, kg, O.BRUTE)
    save("gauss_48x40_s60_b8_k9", "test_baselines.cpp:104-128; matching.cpp:167-182",
         image=img, bins=8, kw=9, sigma=0.6, model_cake=mc, model_brute=mb,
         map_cake=R.likelihood_map(img, 8, mc, kg, O.CAKE, rings=5)[0],
         map_cake_inter=R.likelihood_map(img, 8, mc, kg, O.CAKE, O.INTERSECTION, rings=5)[0],
         map_brute=R.likelihood_map(img, 8, mb, kg, O.BRUTE)[0],
         map_brute_inter=R.likelihood_map(img, 8, mb, kg, O.BRUTE, O.INTERSECTION)[0])

    # 7. ChebyshevLinear (integer, non-affine): brute map; cake with level rule
    img = R.random_gray(40, 36, 5)
    kc = K(O.CHEBYSHEV, 7, 5)
    templ = np.ascontiguousarray(img[3:8, 4:11])
    mdl = R.target_model(templ, 8, kc, O.BRUTE)
    save("cheb_40x36_s5_b8_k7x5", "baselines.cpp:24-51; matching.cpp:175-182", image=img,
         bins=8, model=mdl, map_brute=R.likelihood_map(img, 8, mdl, kc, O.BRUTE)[0],
         map_cake_level=R.likelihood_map(img, 8, mdl, kc, O.CAKE, rings=2, rule=O.RING_LEVEL)[0])

    # 8. C1-like synthetic scene at reduced size (blurred noise + planted patch)
    sc = synth.gray_scene(96, 80, 7, [(21, 21)])
    cx, cy, _, _ = sc.targets[0]
    k = K(O.MANHATTAN, 21, 21)
    templ = synth.crop(sc.image, cx, cy, 21, 21)
    mdl = R.target_model(templ, 16, k)
    mp, pk = R.likelihood_map(sc.image, 16, mdl, k, O.SWIH)
    save("scene_96x80_man21_b16", "acceptance_main.cpp:199-229 (map equivalence) on a synth scene",
         image=sc.image, bins=16, model=mdl, map=mp, peak=np.array(pk),
         target=np.array(sc.targets[0]))

    # 9. a 256x256 C1-shaped case (config 1 generator, 33x33 Manhattan, b=16)
    sc = synth.config1(3)
    cx, cy, _, _ = sc.targets[0]
    k = K(O.MANHATTAN, 33, 33)
    templ = synth.crop(sc.image, cx, cy, 33, 33)
    mdl = R.target_model(templ, 16, k)
    mp, pk = R.likelihood_map(sc.image, 16, mdl, k, O.SWIH, threads=8)
    save("config1_s3", "BASELINE.json configs[0] at full size; matching.cpp:108-223",
         image=sc.image, bins=16, model=mdl, map=mp, peak=np.array(pk),
         target=np.array(sc.targets[0]))

    # 10. tie rule (test_matching.cpp:163-189)
    scores = np.array([[0.2, 0.9, 0.1], [0.9, 0.3, 0.9]])
    save("peak_ties", "test_matching.cpp:163-189", scores=scores,
         peak=np.array(R.peak(scores, 1, 2)))


if __name__ == "__main__":
    main()
