"""Generate tests/golden/golden.npz from the COMPILED REFERENCE (oracle/_ref).

Run in the container where /root/reference exists:
    make -C oracle && python tests/golden/make_golden.py

Every fixture re-expresses a known-answer or oracle test of the reference's
own suite (proj/tests/test_*.cpp, acceptance_main.cpp; cited per block) as
concrete input -> output arrays produced by the reference library itself.
Inputs come from the reference's own generators (tests/synthetic.cpp via
ref_synth); their SHA-256 digests are stored too, so the repo's generator
restatement (paper_2001_07809_b200/synth.py) is pinned against them.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ref = oracle.reference()
    if ref is None:
        raise SystemExit("oracle/_ref/libstk_ref.so missing: build it with make -C oracle")
    S = oracle.ref_synth
    g = {}
    digests = {}

    # ---- lightness (test_imaging.cpp:150-201)
    g["L_endpoints_in"] = np.array([[[0, 0, 0], [255, 255, 255]]], np.uint8)
    g["L_endpoints_out"] = ref.lightness(g["L_endpoints_in"])
    rgb = S("random_rgb", 100, 100, 77)
    digests["random_rgb_100_100_77"] = sha(rgb)
    g["L_random77_out"] = ref.lightness(rgb)
    g["L_dark_in"] = np.array([[[0, 0, 1], [1, 0, 0], [1, 1, 1], [2, 1, 0]]], np.uint8)
    g["L_dark_out"] = ref.lightness(g["L_dark_in"])
    grey = np.repeat(np.arange(256, dtype=np.uint8)[None, :, None], 3, axis=2)
    g["L_grey_axis_out"] = ref.lightness(grey)
    # G2 frame (config A) lightness of both views
    for name, args in [("bench_frame", (200, 150, 7)), ("rectangle_scene", (96, 72, 4, 63)),
                       ("translated_noise", (40, 20, 5, 7))]:
        l, r = S(name, *args)
        digests[f"{name}_{'_'.join(map(str, args))}"] = sha(np.stack([l, r]))

    # ---- histogram + K-Means (test_segmentation.cpp:13-103, acceptance 7a)
    km_c, km_a, km_i = [], [], []
    for seed in range(50):
        img = S("random_gray", 64, 64, 1000 + seed)
        if seed == 0:
            digests["random_gray_64_64_1000"] = sha(img)
        h = ref.histogram(img)
        for k in (2, 4, 10):
            c, a, it = ref.kmeans(h, k)
            cc = np.zeros(10)
            cc[:k] = c
            km_c.append(cc)
            km_a.append(a)
            km_i.append(it)
    g["km_centers"] = np.array(km_c)
    g["km_assign"] = np.array(km_a, np.uint16)
    g["km_iters"] = np.array(km_i, np.int32)
    two = np.array([[10] * 5, [200] * 5], np.uint8)
    c, a, it = ref.kmeans(ref.histogram(two), 2)
    g["km_two_centers"], g["km_two_assign"] = c, a
    g["km_const_hist"] = ref.histogram(np.full((2, 2), 7, np.uint8))

    # ---- boundary detection (test_boundary.cpp:56-66)
    det_in, det_out = [], []
    for seed in range(20):
        words = _raw_words(300 + seed, 32 * 32)
        lab = (words % 3).astype(np.uint16).reshape(32, 32)
        det_in.append(lab)
        det_out.append(ref.detect(lab))
    g["det_in"] = np.array(det_in)
    g["det_out"] = np.array(det_out)

    # ---- fill / remove truth tables (test_boundary.cpp:109-141, acceptance 7c)
    nb = np.array([[(bits >> i) & 1 for i in range(9)] for bits in range(512)], np.uint8)
    g["nb_fill"] = np.array([ref.fill(m.reshape(3, 3)).reshape(9) for m in nb])
    g["nb_remove"] = np.array([ref.remove(m.reshape(3, 3)).reshape(9) for m in nb])
    mf, mr, mp = [], [], []
    for seed in range(20):
        m = S("random_mask", 40, 30, 400 + seed, 35)
        mf.append(ref.fill(m))
        mr.append(ref.remove(m))
        mp.append(ref.prune(m, 0.10))
    g["morph_fill"], g["morph_remove"], g["morph_prune10"] = map(np.array, (mf, mr, mp))
    digests["random_mask_40_30_400_35"] = sha(S("random_mask", 40, 30, 400, 35))

    # ---- connected components (test_boundary.cpp:161-202, acceptance 7b)
    for seed in range(50):
        w = 16 + seed % 49
        h = 8 + (seed * 7) % 57
        m = S("random_mask", w, h, 500 + seed, 30)
        lab, sz, bys = ref.label_components(m)
        g[f"cc{seed}_labels"], g[f"cc{seed}_sizes"], g[f"cc{seed}_bysize"] = lab, sz, bys
    # ---- prune (test_boundary.cpp:204-251)
    pr = []
    for seed in range(20):
        m = S("random_mask", 40, 30, 800 + seed, 20)
        pr.append(ref.prune(m, (seed % 5) * 0.05))
    g["prune_random"] = np.array(pr)
    # ---- anchors (test_boundary.cpp:260-288)
    g["anch_10_4"] = ref.anchors(np.zeros((10, 10), np.uint8), 4)
    g["anch_7_0"] = ref.anchors(np.zeros((5, 7), np.uint8), 0)
    g["anch_rand"] = ref.anchors(S("random_mask", 30, 20, 11, 25), 3)

    # ---- SAD matching (test_stereo.cpp:23-167)
    a = S("random_gray", 24, 18, 5)
    m = S("random_mask", 24, 18, 6, 30)
    g["match_self"] = ref.match(a, a, m, 5, 8)
    l = S("random_gray", 28, 16, 8)
    r = S("random_gray", 28, 16, 9)
    m = S("random_mask", 28, 16, 10, 40)
    g["match_rand"] = ref.match(l, r, m, 3, 7)
    tl, tr = S("translated_noise", 40, 20, 5, 7)
    gl, gr = ref.lightness(tl), ref.lightness(tr)
    g["match_trans"] = ref.match(gl, gr, np.ones((20, 40), np.uint8), 5, 8)
    tl, tr = S("translated_noise", 48, 30, 4, 12)
    gl, gr = ref.lightness(tl), ref.lightness(tr)
    m = S("random_mask", 48, 30, 13, 35)
    g["match_w9"] = ref.match(gl, gr, m, 9, 16)
    img = S("random_gray", 12, 8, 11)
    g["match_edge"] = ref.match(img, img, np.ones((8, 12), np.uint8), 3, 6)

    # ---- reconstruction (test_reconstruct.cpp:31-145, acceptance 7d)
    sp, fi, pk0, pk1 = [], [], [], []
    for seed in range(10):
        s = S("random_sparse", 32, 24, 600 + seed, 12, 15)
        f = ref.fill_scanlines(s)
        sp.append(s)
        fi.append(f)
        pk0.append(ref.peek_columns(f, 0))
        pk1.append(ref.peek_columns(f, 1))
    g["rec_sparse"], g["rec_fill"], g["rec_peek0"], g["rec_peek1"] = map(np.array, (sp, fi, pk0, pk1))
    s = S("random_sparse", 40, 28, 21, 18, 12)
    g["rec_s21"] = s

    # ---- refocus (test_refocus.cpp:23-209, acceptance 7e)
    for sigma, size in ((0.5, 3), (2.0, 13), (8.0, 49), (1.5, 9), (2.0, 9), (1.0, 3)):
        g[f"gk_{sigma}_{size}"] = ref.gaussian_kernel(sigma, size)
    dm = np.array([[2, 4, 11, 7]], np.int16)
    g["bm_simple"] = ref.blur_map(dm, [(3, 5), (10, 12)], 16)
    img = S("random_rgb", 21, 15, 43)
    msk = S("random_mask", 21, 15, 44, 50)
    g["blur_sharp_next"] = ref.selective_blur(img, msk, 2.0, 9)
    img = S("random_rgb", 33, 27, 45)
    msk = S("random_mask", 33, 27, 46, 40)
    g["blur_rand"] = ref.selective_blur(img, msk, 2.0, 9)
    edge = np.zeros((3, 3, 3), np.uint8)
    edge[0, 0] = 255
    g["blur_edge"] = ref.selective_blur(edge, np.ones((3, 3), np.uint8), 1.0, 3)

    # ---- whole pipeline (test_pipeline.cpp:48-168, acceptance 5 and 8)
    def frame(tag, l, r, **kw):
        res = ref.run_frame(l, r, **kw)
        for k in ("dense", "sparse", "left_lightness", "labels", "boundary_raw", "boundary_refined",
                  "boundary_anchored", "row_filled", "refocused"):
            if res.get(k) is not None:
                g[f"{tag}_{k}"] = res[k]
        g[f"{tag}_centers"] = res["centers"]
        g[f"{tag}_kit"] = np.array([res["k"], res["iterations_run"]], np.int32)
        st = res["stats"]
        g[f"{tag}_stats"] = np.array([st["pixels"], st["boundary_raw"], st["boundary_refined"],
                                      st["matched"]], np.int64)

    l, r = S("rectangle_scene", 96, 72, 4, 63)
    frame("pipe_rect", l, r, k=2, max_disparity=8, focus=[(3, 8)])
    l, r = S("rectangle_scene", 96, 72, 0, 60)
    frame("pipe_self", l, l, k=2, max_disparity=8)
    for i in range(20):
        l, r = S("translated_noise", 128, 96, i % 9, 500 + i)
        frame(f"crit5_{i}", l, r, k=10, max_disparity=12, focus=[(2, 6)], sigma=1.5)
    for s in range(1, 9):
        l, r = S("rectangle_scene", 160, 120, s, 700 + s)
        frame(f"crit8_{s}", l, r, k=2, window=9, max_disparity=16)
    # the benchmark's own scene (G2 dead leaves, config A) through the reference
    from paper_2001_07809_b200 import synth

    l, r = synth.dead_leaves(450, 375, 16, frame=0)
    digests["dead_leaves_450_375_16_0"] = sha(np.stack([l, r]))
    frame("g2A", l, r, k=4, window=9, max_disparity=16, focus=[(8, 16)], sigma=2.0)
    l, r = S("bench_frame", 200, 150, 7)
    frame("g1", l, r, k=10, window=9, max_disparity=16, focus=[(8, 16)], sigma=2.0)

    g["digest_keys"] = np.array(sorted(digests))
    g["digest_vals"] = np.array([digests[k] for k in sorted(digests)])
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


def _raw_words(seed, n):
    """std::mt19937(seed) raw draws (test_boundary.cpp:26-33 random_labels).  The
    reference exposes raw draws only inside its generators, so this uses the
    repo's engine, which test_oracle_cpu.py pins against those generators."""
    from paper_2001_07809_b200 import synth

    out = np.empty(n, np.uint32)
    synth._raw_words(seed, out)
    return out


if __name__ == "__main__":
    main()
