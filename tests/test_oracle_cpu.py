"""CPU-only tests: pin the oracle (C restatement) and the synthetic generators
against the golden fixtures made by the compiled reference, cross-check the
oracle against the compiled reference when present, verify the L* threshold
rule over all 2^24 RGB triples, and check the C-ABI library surface (symbols,
host-only entries, loud failure without a GPU)."""
import ctypes as C
import hashlib
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ------------------------------------------------------------- generators --
def test_generators_match_reference_digests(golden, synth):
    dig = dict(zip(golden["digest_keys"], golden["digest_vals"]))
    assert dig["random_rgb_100_100_77"] == sha(synth.random_rgb(100, 100, 77))
    assert dig["random_gray_64_64_1000"] == sha(synth.random_gray(64, 64, 1000))
    assert dig["random_mask_40_30_400_35"] == sha(synth.random_mask(40, 30, 400, 35))
    assert dig["bench_frame_200_150_7"] == sha(np.stack(synth.bench_frame(200, 150, 7)))
    assert dig["rectangle_scene_96_72_4_63"] == sha(np.stack(synth.rectangle_scene_pair(96, 72, 4, 63)))
    assert dig["translated_noise_40_20_5_7"] == sha(np.stack(synth.translated_noise_pair(40, 20, 5, 7)))
    assert dig["dead_leaves_450_375_16_0"] == sha(np.stack(synth.dead_leaves(450, 375, 16, frame=0)))


def test_generators_match_compiled_reference(ref, synth):
    import oracle

    for args in ((200, 150, 7), (97, 61, 3)):
        a = oracle.ref_synth("bench_frame", *args)
        b = synth.bench_frame(*args)
        assert all((x == y).all() for x, y in zip(a, b))
    for args in ((96, 72, 4, 63), (160, 120, 8, 708)):
        a = oracle.ref_synth("rectangle_scene", *args)
        assert all((x == y).all() for x, y in zip(a, synth.rectangle_scene_pair(*args)))
    a = oracle.ref_synth("translated_noise", 128, 96, 5, 505)
    assert all((x == y).all() for x, y in zip(a, synth.translated_noise_pair(128, 96, 5, 505)))
    assert (oracle.ref_synth("random_sparse", 32, 24, 600, 12, 15) ==
            synth.random_sparse(32, 24, 600, 12, 15)).all()


def test_dead_leaves_density_matches_survey(port, synth):
    """config A / K4 -> matched 17.9 %, known 98.2 %, 11 iterations."""
    l, r = synth.dead_leaves(450, 375, 16, frame=0)
    res = port.run_frame(l, r, k=4, window=9, max_disparity=16)
    assert round(res["stats"]["matched_fraction"] * 100, 1) == 17.9
    assert round(res["stats"]["known_fraction"] * 100, 1) == 98.2
    assert res["iterations_run"] == 11


# --------------------------------------------------- oracle vs golden ------
def test_oracle_lightness_golden(golden, port, synth):
    assert (port.lightness(golden["L_endpoints_in"]) == golden["L_endpoints_out"]).all()
    assert (port.lightness(synth.random_rgb(100, 100, 77)) == golden["L_random77_out"]).all()
    assert (port.lightness(golden["L_dark_in"]) == golden["L_dark_out"]).all()
    grey = np.repeat(np.arange(256, dtype=np.uint8)[None, :, None], 3, axis=2)
    out = port.lightness(grey)
    assert (out == golden["L_grey_axis_out"]).all()
    assert out[0, 0] == 0 and out[0, 255] == 255 and (np.diff(out[0].astype(int)) >= 0).all()
    assert 134 <= port.lightness(np.full((1, 1, 3), 128, np.uint8))[0, 0] <= 139


def test_oracle_kmeans_golden(golden, port, synth):
    i = 0
    for seed in range(50):
        h = port.histogram(synth.random_gray(64, 64, 1000 + seed))
        for k in (2, 4, 10):
            c, a, it = port.kmeans(h, k)
            assert (c == golden["km_centers"][i][:k]).all()
            assert (a == golden["km_assign"][i]).all()
            assert it == golden["km_iters"][i]
            i += 1
    c, a, _ = port.kmeans(port.histogram(np.array([[10] * 5, [200] * 5], np.uint8)), 2)
    assert (c == golden["km_two_centers"]).all() and (a == golden["km_two_assign"]).all()


def test_oracle_boundary_golden(golden, port, synth):
    for lab, want in zip(golden["det_in"], golden["det_out"]):
        assert (port.detect(lab) == want).all()
    nb = np.array([[(b >> i) & 1 for i in range(9)] for b in range(512)], np.uint8)
    for m, wf, wr in zip(nb, golden["nb_fill"], golden["nb_remove"]):
        assert (port.fill(m.reshape(3, 3)).reshape(9) == wf).all()
        assert (port.remove(m.reshape(3, 3)).reshape(9) == wr).all()
    for s in range(20):
        m = synth.random_mask(40, 30, 400 + s, 35)
        assert (port.fill(m) == golden["morph_fill"][s]).all()
        assert (port.remove(m) == golden["morph_remove"][s]).all()
        assert (port.prune(m, 0.10) == golden["morph_prune10"][s]).all()


def test_oracle_components_golden(golden, port, synth):
    for seed in range(50):
        w, h = 16 + seed % 49, 8 + (seed * 7) % 57
        lab, sz, bys = port.label_components(synth.random_mask(w, h, 500 + seed, 30))
        assert (lab == golden[f"cc{seed}_labels"]).all()
        assert (sz == golden[f"cc{seed}_sizes"]).all()
        assert (bys == golden[f"cc{seed}_bysize"]).all()
    for s in range(20):
        m = synth.random_mask(40, 30, 800 + s, 20)
        assert (port.prune(m, (s % 5) * 0.05) == golden["prune_random"][s]).all()
    assert (port.anchors(np.zeros((10, 10), np.uint8), 4) == golden["anch_10_4"]).all()
    assert (port.anchors(np.zeros((5, 7), np.uint8), 0) == golden["anch_7_0"]).all()
    assert (port.anchors(synth.random_mask(30, 20, 11, 25), 3) == golden["anch_rand"]).all()


def test_oracle_match_golden(golden, port, synth):
    a = synth.random_gray(24, 18, 5)
    assert (port.match(a, a, synth.random_mask(24, 18, 6, 30), 5, 8) == golden["match_self"]).all()
    l, r = synth.random_gray(28, 16, 8), synth.random_gray(28, 16, 9)
    assert (port.match(l, r, synth.random_mask(28, 16, 10, 40), 3, 7) == golden["match_rand"]).all()
    tl, tr = synth.translated_noise_pair(48, 30, 4, 12)
    gl, gr = port.lightness(tl), port.lightness(tr)
    assert (port.match(gl, gr, synth.random_mask(48, 30, 13, 35), 9, 16) == golden["match_w9"]).all()


def test_oracle_reconstruct_golden(golden, port):
    for s, f, p0, p1 in zip(golden["rec_sparse"], golden["rec_fill"], golden["rec_peek0"],
                            golden["rec_peek1"]):
        assert (port.fill_scanlines(s) == f).all()
        assert (port.peek_columns(f, 0) == p0).all()
        assert (port.peek_columns(f, 1) == p1).all()


def test_oracle_refocus_golden(golden, port, synth):
    for sigma, size in ((0.5, 3), (2.0, 13), (8.0, 49), (1.5, 9)):
        assert (port.gaussian_kernel(sigma, size) == golden[f"gk_{sigma}_{size}"]).all()
    img, msk = synth.random_rgb(33, 27, 45), synth.random_mask(33, 27, 46, 40)
    assert (port.selective_blur(img, msk, 2.0, 9) == golden["blur_rand"]).all()


@pytest.mark.parametrize("tag", ["pipe_rect", "crit5_3", "crit8_5", "g2A", "g1"])
def test_oracle_pipeline_golden(golden, port, synth, tag):
    if tag == "pipe_rect":
        l, r = synth.rectangle_scene_pair(96, 72, 4, 63)
        kw = dict(k=2, max_disparity=8, focus=[(3, 8)])
    elif tag.startswith("crit5"):
        i = int(tag.split("_")[1])
        l, r = synth.translated_noise_pair(128, 96, i % 9, 500 + i)
        kw = dict(k=10, max_disparity=12, focus=[(2, 6)], sigma=1.5)
    elif tag.startswith("crit8"):
        s = int(tag.split("_")[1])
        l, r = synth.rectangle_scene_pair(160, 120, s, 700 + s)
        kw = dict(k=2, window=9, max_disparity=16)
    elif tag == "g2A":
        l, r = synth.dead_leaves(450, 375, 16, frame=0)
        kw = dict(k=4, window=9, max_disparity=16, focus=[(8, 16)], sigma=2.0)
    else:
        l, r = synth.bench_frame(200, 150, 7)
        kw = dict(k=10, window=9, max_disparity=16, focus=[(8, 16)], sigma=2.0)
    res = port.run_frame(l, r, **kw)
    for k in ("dense", "sparse", "left_lightness", "labels", "boundary_raw", "boundary_refined",
              "boundary_anchored", "row_filled", "refocused"):
        key = f"{tag}_{k}"
        if key in golden.files:
            assert (res[k] == golden[key]).all(), k


# --------------------------------------- oracle vs compiled reference ------
def test_oracle_matches_reference_random(ref, port, synth):
    rng = np.random.default_rng(7)
    for t in range(6):
        w, h = int(rng.integers(5, 90)), int(rng.integers(5, 70))
        rgb = synth.random_rgb(w, h, 9000 + t)
        assert (port.lightness(rgb) == ref.lightness(rgb)).all()
        m = synth.random_mask(w, h, 9100 + t, int(rng.integers(5, 70)))
        assert (port.fill(m) == ref.fill(m)).all() and (port.remove(m) == ref.remove(m)).all()
        a, b = port.label_components(m), ref.label_components(m)
        assert all((x == y).all() for x, y in zip(a, b))
        for frac in (0.0, 0.04, 0.3):
            assert (port.prune(m, frac) == ref.prune(m, frac)).all()
        s = synth.random_sparse(w, h, 9200 + t, int(rng.integers(3, 60)), 20)
        f = port.fill_scanlines(s)
        assert (f == ref.fill_scanlines(s)).all()
        for thr in (0, 1, 3):
            assert (port.peek_columns(f, thr) == ref.peek_columns(f, thr)).all()


def test_oracle_pipeline_matches_reference_g1(ref, port, synth):
    l, r = synth.dead_leaves(160, 120, 12, frame=3)
    a = port.run_frame(l, r, k=5, window=7, max_disparity=12, focus=[(0, 4), (9, 12)], sigma=1.2)
    b = ref.run_frame(l, r, k=5, window=7, max_disparity=12, focus=[(0, 4), (9, 12)], sigma=1.2)
    for k in ("dense", "sparse", "labels", "boundary_anchored", "refocused"):
        assert (a[k] == b[k]).all(), k


# ------------------------------------------------ L* threshold rule (2^24) --
def test_lstar_threshold_rule_exhaustive(port):
    """gray(Y) = #{v : thr[v] <= Y} equals the reference formula for every RGB
    triple -- the rule K1 evaluates on the device (no device cbrt/pow)."""
    from paper_2001_07809_b200 import _lib

    lin = np.zeros(256)
    thr = np.zeros(256)
    _lib.lib().stk_lstar_tables(lin.ctypes.data_as(C.c_void_p), thr.ctypes.data_as(C.c_void_p))
    assert thr[0] == -1.0 and (np.diff(thr[1:]) > 0).all()
    v = np.arange(256)
    rgb = np.stack(np.meshgrid(v, v, v, indexing="ij"), -1).reshape(4096, 4096, 3).astype(np.uint8)
    want = port.lightness(rgb).reshape(-1)
    r, g, b = (rgb.reshape(-1, 3)[:, i] for i in range(3))
    # same association and rounding as lightness.cpp:41-43 (numpy float64, no FMA)
    y = (0.2126 * lin[r] + 0.7152 * lin[g]) + 0.0722 * lin[b]
    got = np.searchsorted(thr[1:], y, side="right")
    assert (got == want).all()


# -------------------------------------------------------- C-ABI surface ----
def test_abi_exports_every_declared_symbol():
    from paper_2001_07809_b200 import _lib

    hdr = open(os.path.join(ROOT, "include", "stk_b200.h")).read()
    names = set(re.findall(r"\b(stk_[a-z0-9_]+)\s*\(", hdr))
    L = _lib.lib()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert names <= set(_lib.SIGNATURES), names - set(_lib.SIGNATURES)
    assert L.stk_abi_version() == 1


def test_host_only_entries_match_reference(port, stk):
    for s in (0.5, 1.0, 2.0, 2.5, 8.0):
        assert stk.default_kernel_size(s) == port.lib.orc_default_kernel_size(s)
    for sigma, size in ((0.5, 3), (2.0, 13), (8.0, 49)):
        assert (stk.gaussian_kernel(sigma, size).weights == port.gaussian_kernel(sigma, size)).all()
    with pytest.raises(stk.ParamError):
        stk.gaussian_kernel(0.0, 3)
    with pytest.raises(stk.ParamError):
        stk.gaussian_kernel(1.0, 4)
    stk.validate_config(stk.PipelineConfig())
    for bad in (dict(window=4), dict(k=0), dict(threshold=-1), dict(prune_fraction=1.0),
                dict(workers=0), dict(max_disparity=-1)):
        with pytest.raises(stk.ParamError):
            stk.validate_config(stk.PipelineConfig(**bad))


def test_no_gpu_fails_loudly(stk):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(stk.CudaError, match="no CUDA device"):
        stk.Device(0)


def test_port_evaluation_matches_reference(ref, port):
    """The port's bad_pixel_rate / dense_sad_baseline restatements equal the
    compiled reference (evaluate.cpp)."""
    rng = np.random.default_rng(77)
    for (w, h) in ((16, 12), (50, 40), (97, 33)):
        a = rng.integers(-1, 30, (h, w)).astype(np.int16)
        b = rng.integers(-1, 30, (h, w)).astype(np.int16)
        for d in (0.0, 1.0, 2.5):
            assert port.bad_pixel_rate(a, b, d)[:3] == ref.bad_pixel_rate(a, b, d)[:3]
        l = rng.integers(0, 255, (h, w), dtype=np.uint8)
        r = np.roll(l, -2, axis=1)
        for win, D in ((3, 6), (5, 16), (9, 4)):
            np.testing.assert_array_equal(port.dense_sad_baseline(l, r, win, D),
                                          ref.dense_sad_baseline(l, r, win, D))
