"""GPU parity, stage by stage: every C-ABI stage entry (through the Python
mirror of the stereotk API) against the golden fixtures of the compiled
reference and against the oracle on seeded random inputs, including the
reference suite's edge cases.  Bit-exact everywhere except the separable
blur (<= 1 LSB, tolerance written below)."""
import os
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BLUR_TOL_LSB = 1  # north star: blurred 8-bit output within <= 1 LSB


def eq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    bad = int((a != b).sum())
    assert bad == 0, f"{bad} mismatching elements"


# ----------------------------------------------------------------- K1 -------
def test_lightness_golden(dev, stk, golden, synth):
    eq(stk.rgb_to_lightness(golden["L_endpoints_in"], device=dev), golden["L_endpoints_out"])
    eq(stk.rgb_to_lightness(synth.random_rgb(100, 100, 77), device=dev), golden["L_random77_out"])
    eq(stk.rgb_to_lightness(golden["L_dark_in"], device=dev), golden["L_dark_out"])
    grey = np.repeat(np.arange(256, dtype=np.uint8)[None, :, None], 3, axis=2)
    eq(stk.rgb_to_lightness(grey, device=dev), golden["L_grey_axis_out"])


def test_lightness_all_2pow24_triples(dev, stk, port):
    v = np.arange(256)
    rgb = np.stack(np.meshgrid(v, v, v, indexing="ij"), -1).reshape(4096, 4096, 3).astype(np.uint8)
    eq(stk.rgb_to_lightness(rgb, device=dev), port.lightness(rgb))


@pytest.mark.parametrize("w,h", [(1, 1), (3, 2), (17, 5), (450, 375), (1000, 3)])
def test_lightness_and_histogram_ragged(dev, stk, port, synth, w, h):
    rgb = synth.random_rgb(w, h, 11 * w + h)
    g = stk.rgb_to_lightness(rgb, device=dev)
    eq(g, port.lightness(rgb))
    eq(stk.build_histogram(g, device=dev), port.histogram(g))


# ----------------------------------------------------------------- K2 -------
def test_kmeans_golden(dev, stk, golden, synth):
    i = 0
    for seed in range(50):
        img = synth.random_gray(64, 64, 1000 + seed)
        h = stk.build_histogram(img, device=dev)
        for k in (2, 4, 10):
            c = stk.kmeans_histogram(h, k, device=dev)
            assert (c.centers == golden["km_centers"][i][:k]).all()  # exact FP64 equality
            eq(c.bin_assignment, golden["km_assign"][i])
            assert c.iterations_run == golden["km_iters"][i]
            i += 1


def test_kmeans_edge_cases(dev, stk, port):
    two = np.array([[10] * 5, [200] * 5], np.uint8)
    c = stk.kmeans_histogram(stk.build_histogram(two, device=dev), 2, device=dev)
    assert list(c.centers) == [10.0, 200.0]
    labels = stk.assign_pixels(two, c, device=dev)
    assert (labels[0] == 0).all() and (labels[1] == 1).all()
    one = np.full((3, 3), 42, np.uint8)
    assert stk.kmeans_histogram(stk.build_histogram(one, device=dev), 1, device=dev).centers[0] == 42.0
    h = stk.build_histogram(np.array([[1, 2, 3, 4]], np.uint8), device=dev)
    for k, it in ((0, 100), (-3, 100), (5, 100), (2, 0)):
        with pytest.raises(stk.ParamError):
            stk.kmeans_histogram(h, k, it, device=dev)
    with pytest.raises(stk.ParamError, match="empty histogram"):
        stk.kmeans_histogram(np.zeros(256, np.uint64), 1, device=dev)
    # many clusters, odd max_iter / tol, against the oracle
    rng = np.random.default_rng(3)
    for t in range(10):
        counts = (rng.integers(0, 5, 256) * rng.integers(0, 1000, 256)).astype(np.uint64)
        occ = int((counts > 0).sum())
        for k in (1, min(occ, 37), occ):
            want = port.kmeans(counts, k, 7 + t, 0.25 * t)
            got = stk.kmeans_histogram(counts, k, 7 + t, 0.25 * t, device=dev)
            assert (got.centers == want[0]).all() and (got.bin_assignment == want[1]).all()
            assert got.iterations_run == want[2]


# ----------------------------------------------------------------- K3 -------
def test_detect_golden(dev, stk, golden):
    for lab, want in zip(golden["det_in"], golden["det_out"]):
        eq(stk.detect_boundaries(lab, device=dev), want)


def test_detect_fill_remove_edge_cases(dev, stk, port, synth):
    assert stk.detect_boundaries(np.zeros((6, 8), np.uint16), device=dev).sum() == 0
    lab = np.zeros((4, 8), np.uint16)
    lab[:, 3:] = 1
    m = stk.detect_boundaries(lab, device=dev)
    assert (m[:, 2] == 1).all() and (m[:, 3] == 1).all() and m.sum() == 8
    nb = np.array([[(b >> i) & 1 for i in range(9)] for b in range(512)], np.uint8)
    for bits in range(512):
        mm = nb[bits].reshape(3, 3)
        eq(stk.morph_fill(mm, device=dev), port.fill(mm))
        eq(stk.morph_remove(mm, device=dev), port.remove(mm))
    for w, h in ((1, 1), (2, 7), (3, 3), (129, 33), (300, 65), (64, 1)):
        m = synth.random_mask(w, h, w * 7 + h, 60)
        eq(stk.morph_fill(m, device=dev), port.fill(m))
        eq(stk.morph_remove(m, device=dev), port.remove(m))
        lab = (synth.random_gray(w, h, w + h) % 3).astype(np.uint16)
        eq(stk.detect_boundaries(lab, device=dev), port.detect(lab))


def test_detect_fill_remove_hot_path_kernel_cases(dev, stk, port, synth):
    """The stage entries run the frame path's B1 kernel (k_morph_bits in stage
    mode).  Cases beyond the frame's own inputs: 16-bit labels above 255 (the
    second bit-plane pass), label pairs differing only in high bits, mask
    bytes other than 0/1 (the reference copies them through, boundary.cpp:42,
    :66), widths around the 32-pixel word and the 30-word warp strip, and
    heights around the 8-row band."""
    rng = np.random.default_rng(7)
    for w, h in ((31, 9), (32, 8), (33, 17), (959, 7), (960, 16), (961, 3), (1000, 41)):
        lab = rng.integers(0, 65536, size=(h, w), dtype=np.uint16)
        lab[: h // 2] = lab[: h // 2] & 0xFF00  # blocks equal in the low byte
        lab[:, ::7] = 0x8000
        eq(stk.detect_boundaries(lab, device=dev), port.detect(lab))
        lab2 = (synth.random_gray(w, h, w * h) % 2).astype(np.uint16) * 0x0100  # only bit 8 differs
        eq(stk.detect_boundaries(lab2, device=dev), port.detect(lab2))
        m = synth.random_mask(w, h, w + 3 * h, 70)
        m = m * rng.choice(np.array([1, 2, 255], np.uint8), size=m.shape)
        eq(stk.morph_fill(m, device=dev), port.fill(m))
        eq(stk.morph_remove(m, device=dev), port.remove(m))


def test_morph_golden(dev, stk, golden, synth):
    for s in range(20):
        m = synth.random_mask(40, 30, 400 + s, 35)
        eq(stk.morph_fill(m, device=dev), golden["morph_fill"][s])
        eq(stk.morph_remove(m, device=dev), golden["morph_remove"][s])


# ----------------------------------------------------------------- K4 -------
def test_components_golden(dev, stk, golden, synth):
    for seed in range(50):
        w, h = 16 + seed % 49, 8 + (seed * 7) % 57
        t = stk.label_components(synth.random_mask(w, h, 500 + seed, 30), device=dev)
        eq(t.labels, golden[f"cc{seed}_labels"])
        eq(t.sizes, golden[f"cc{seed}_sizes"])
        eq(t.by_size, golden[f"cc{seed}_bysize"])


@pytest.mark.parametrize("w,h,pct", [(1, 1, 100), (5, 200, 50), (333, 77, 30), (1024, 96, 12),
                                     (2000, 40, 45), (97, 1, 60)])
def test_components_and_prune_random(dev, stk, port, synth, w, h, pct):
    m = synth.random_mask(w, h, 31 * w + h, pct)
    t = stk.label_components(m, device=dev)
    lab, sz, bys = port.label_components(m)
    eq(t.labels, lab)
    eq(t.sizes, sz)
    eq(t.by_size, bys)
    for frac in (0.0, 0.04, 0.1, 0.5, 0.999):
        eq(stk.prune_components(m, frac, device=dev), port.prune(m, frac))


@pytest.mark.parametrize("case", ["random_1080p", "comb", "frame_mask"])
def test_components_run_ccl_large(dev, stk, port, synth, case):
    """label_components on the frame path's run CCL (B2 region merge, B3
    global union, label kernels): large masks crossing many 256x128 regions,
    one giant component, and a real frame's refined boundary mask."""
    if case == "random_1080p":
        m = synth.random_mask(1920, 1080, 99, 45)
    elif case == "comb":
        m = np.zeros((300, 700), np.uint8)
        m[5, :] = 1
        m[5:290, ::31] = 1
        m[63:65, :600] = 1
        m[100:300:4, 3:700:5] = 1
        m[31:33, 127:129] = 1
    else:
        l, r = synth.dead_leaves(1024, 576, 32, frame=3)
        res = port.run_frame(l, r, k=6, window=9, max_disparity=32)
        m = res["boundary_refined"]
    t = stk.label_components(m, device=dev)
    lab, sz, bys = port.label_components(m)
    eq(t.labels, lab)
    eq(t.sizes, sz)
    eq(t.by_size, bys)


def test_components_and_prune_repeated_large(dev, stk, port, synth):
    """Repeated large masks (the compress passes run concurrently with no
    ordering between threads): labels, sizes, by_size and the pruned mask equal
    the oracle on every run."""
    for seed in range(6):
        m = synth.random_mask(1920, 1080, 1000 + seed, 40 + seed)
        t = stk.label_components(m, device=dev)
        lab, sz, bys = port.label_components(m)
        eq(t.labels, lab)
        eq(t.sizes, sz)
        eq(t.by_size, bys)
        eq(stk.prune_components(m, 0.04, device=dev), port.prune(m, 0.04))


def test_components_overflow_tiles(dev, stk, port, synth):
    """B2 keeps 224 runs per 32x32 tile in shared memory; regions with a
    denser tile go through the 512-run overflow pass.  Checkerboard rows (16
    runs per row: every tile overflows), a mask where only some regions
    overflow, and a dense random mask: labels, sizes, by_size and the pruned
    mask equal the oracle."""
    W, H = 700, 300
    yy, xx = np.mgrid[0:H, 0:W]
    checker = (((xx + (yy // 3)) % 2) == 0).astype(np.uint8)          # all tiles > 256 runs
    mixed = synth.random_mask(W, H, 5, 20)
    mixed[64:192, 128:384] = checker[64:192, 128:384]                 # a block of overflow regions
    dense = synth.random_mask(W, H, 6, 50)
    for m in (checker, mixed, dense):
        t = stk.label_components(m, device=dev)
        lab, sz, bys = port.label_components(m)
        eq(t.labels, lab)
        eq(t.sizes, sz)
        eq(t.by_size, bys)
        for frac in (0.0, 0.04, 0.3):
            eq(stk.prune_components(m, frac, device=dev), port.prune(m, frac))


def test_components_overflow_pass_loops(dev, stk, port):
    """The overflow pass runs on two CTAs, so each loops over many listed
    regions reusing its shared-memory tables: a 1536x768 checkerboard-row mask
    (every one of its 36 regions overflows), three times."""
    W, H = 1536, 768
    yy, xx = np.mgrid[0:H, 0:W]
    m = (((xx + (yy // 3)) % 2) == 0).astype(np.uint8)
    m[::7, :] = 1                                       # long runs joining the columns
    lab, sz, bys = port.label_components(m)
    pr = port.prune(m, 0.04)
    for _ in range(3):
        t = stk.label_components(m, device=dev)
        eq(t.labels, lab)
        eq(t.sizes, sz)
        eq(t.by_size, bys)
        eq(stk.prune_components(m, 0.04, device=dev), pr)


def test_components_many_region_roots(dev, stk, port):
    """B3 lists the border unions for B3b's shared-memory forest only up to
    32768 region roots; above that it unites them on the global forest.  A
    mask of isolated pixels (196 K region roots) crossed by lines that chain
    them across every region border: labels, sizes, by_size, pruned masks."""
    W, H = 1024, 768
    m = np.zeros((H, W), np.uint8)
    m[::2, ::2] = 1
    m[1::96, :] = 1                      # joins rows 0/2 (and 96/98 ...) across regions
    m[:, 127::128] = 1                   # vertical lines on region edges
    m[300:700, 400:800:3] = 1            # vertical runs crossing region rows
    t = stk.label_components(m, device=dev)
    lab, sz, bys = port.label_components(m)
    eq(t.labels, lab)
    eq(t.sizes, sz)
    eq(t.by_size, bys)
    for frac in (0.0, 0.04, 0.3):
        eq(stk.prune_components(m, frac, device=dev), port.prune(m, frac))


_UNITE_CAP_SNIPPET = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2001_07809_b200 import stereotk as stk, synth
import oracle
port = oracle.port()
d = stk.Device(0, slots=1)
for seed, (w, h, pct) in enumerate([(1920, 1080, 40), (700, 300, 20), (517, 331, 30), (4096, 160, 12)]):
    m = synth.random_mask(w, h, 70 + seed, pct)
    t = stk.label_components(m, device=d)
    lab, sz, bys = port.label_components(m)
    assert np.array_equal(t.labels, lab) and np.array_equal(t.sizes, sz) and np.array_equal(t.by_size, bys), seed
    for frac in (0.0, 0.04, 0.3):
        assert np.array_equal(stk.prune_components(m, frac, device=d), port.prune(m, frac)), (seed, frac)
d.close()
print("ok")
"""


@pytest.mark.parametrize("cap", ["0", "100"])
def test_components_unite_cap(cap, tmp_path):
    """B3's two union paths against the oracle in a fresh process: cap 0 (every
    union on the global forest, no B3b) and cap 100 (small masks through B3b's
    shared-memory forest, large ones directly)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, STK_UNITE_CAP=cap)
    r = subprocess.run([sys.executable, "-c", _UNITE_CAP_SNIPPET, root], capture_output=True, text=True,
                       timeout=600, env=env)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]


def test_prune_golden_and_spec(dev, stk, golden, synth):
    for s in range(20):
        m = synth.random_mask(40, 30, 800 + s, 20)
        eq(stk.prune_components(m, (s % 5) * 0.05, device=dev), golden["prune_random"][s])
    # sizes {1, 2, 97} at 4 % (test_boundary.cpp:204-235)
    m = np.zeros((16, 24), np.uint8)
    m[0:10, 0:10] = 1
    m[9, 9] = m[9, 8] = m[8, 9] = 0
    m[14, 15] = 1
    m[3, 20] = m[3, 21] = 1
    p = stk.prune_components(m, 0.04, device=dev)
    assert p.sum() == 97 and p[14, 15] == 0 and p[3, 20] == 0 and p[0, 0] == 1
    solo = np.zeros((6, 6), np.uint8)
    solo[2, 2] = solo[2, 3] = 1
    assert stk.prune_components(solo, 0.9, device=dev).sum() == 2
    for bad in (-0.1, 1.0, 1.5):
        with pytest.raises(stk.ParamError):
            stk.prune_components(solo, bad, device=dev)


def test_prune_many_equal_sizes_partial_class(dev, stk, port):
    """Ties at the cut size: the first q size-s* components in label order go."""
    m = np.zeros((64, 256), np.uint8)
    m[::3, ::3] = 1  # 22 x 86 isolated pixels: all size 1
    m[60:64, 200:256] = 1  # one big component
    for frac in (0.01, 0.05, 0.2, 0.5):
        eq(stk.prune_components(m, frac, device=dev), port.prune(m, frac))


def test_prune_select_fallbacks(dev, stk, port):
    """B3b does the prune's s*/q select and size classes itself when s* <= 4096
    and at most 2048 components have size s*; otherwise the cooperative prune
    does.  Large blobs only (s* beyond 4096 at high fractions), 3600 equal
    singletons (a size-s* class too long for B3b's list when q > 0), and the
    in-CTA cases next to them."""
    blobs = np.zeros((768, 1024), np.uint8)
    for j in range(12):
        y, x = 40 + 240 * (j // 4), 30 + 250 * (j % 4)
        blobs[y:y + 90 + 5 * j, x:x + 100 + 7 * j] = 1     # 9000 .. 25000 pixels each
    single = np.zeros((480, 640), np.uint8)
    single[::8, ::8] = 1                                   # 4800 isolated pixels
    single[200:260, 300:420] = 1                           # and one blob
    few = np.zeros((480, 640), np.uint8)
    few[::16, ::16] = 1                                    # 1200 singletons: the in-CTA list
    few[100:140, 100:300] = 1
    for m in (blobs, single, few):
        for frac in (0.0, 0.01, 0.2, 0.5, 0.9):
            eq(stk.prune_components(m, frac, device=dev), port.prune(m, frac))


@pytest.mark.parametrize("w,h,seed,pct", [(300, 200, 1, 15), (517, 331, 2, 30), (1024, 256, 3, 8),
                                         (129, 65, 4, 45), (700, 140, 5, 22)])
def test_prune_bitpacked_vs_oracle(dev, stk, port, synth, w, h, seed, pct):
    """prune_components runs the frame path's bit-packed run CCL (region merge
    across 256x128 regions, global union-find, s*/q select, first-q bitmap scan):
    random masks with many small components, crossing tile and region borders,
    at fractions that cut inside a size class (q > 0) and beyond."""
    m = synth.random_mask(w, h, seed, pct)
    for frac in (0.0, 0.01, 0.04, 0.1, 0.3, 0.6):
        eq(stk.prune_components(m, frac, device=dev), port.prune(m, frac))


def test_prune_bitpacked_giant_and_lines(dev, stk, port):
    """One component spanning every region (a comb) next to many singletons and
    2-pixel dominoes, plus long runs along tile / region borders."""
    m = np.zeros((300, 700), np.uint8)
    m[5, :] = 1                      # spine across all regions
    m[5:290:1, ::31] = 1             # teeth down tile borders (x = 0, 31, 62, ...)
    m[63:65, :600] = 1               # a run pair straddling the 64-row region seam
    m[100:300:4, 3:700:5] = 1        # singletons
    m[102:300:8, 1:690:7] = 1
    m[102:300:8, 2:690:7] = 1        # dominoes
    m[31:33, 127:129] = 1            # 2x2 block on a region corner
    for frac in (0.0, 0.02, 0.05, 0.2):
        eq(stk.prune_components(m, frac, device=dev), port.prune(m, frac))


def test_anchors(dev, stk, golden, synth):
    eq(stk.add_border_anchors(np.zeros((10, 10), np.uint8), 4, device=dev), golden["anch_10_4"])
    eq(stk.add_border_anchors(np.zeros((5, 7), np.uint8), 0, device=dev), golden["anch_7_0"])
    eq(stk.add_border_anchors(synth.random_mask(30, 20, 11, 25), 3, device=dev), golden["anch_rand"])
    with pytest.raises(stk.ParamError):
        stk.add_border_anchors(np.zeros((10, 10), np.uint8), -1, device=dev)
    with pytest.raises(stk.ParamError):
        stk.add_border_anchors(np.zeros((10, 10), np.uint8), 5, device=dev)


# ----------------------------------------------------------------- K5 -------
@pytest.fixture(params=["ws", "strip", "list"])
def sad_dev(request, dev):
    dev.set_sad_kernel(request.param)
    yield dev
    dev.set_sad_kernel("auto")


def test_match_golden(sad_dev, stk, golden, synth, port):
    d = sad_dev
    a = synth.random_gray(24, 18, 5)
    eq(stk.match_boundary_pixels(a, a, synth.random_mask(24, 18, 6, 30), stk.MatchConfig(5, 8),
                                 device=d), golden["match_self"])
    l, r = synth.random_gray(28, 16, 8), synth.random_gray(28, 16, 9)
    eq(stk.match_boundary_pixels(l, r, synth.random_mask(28, 16, 10, 40), stk.MatchConfig(3, 7),
                                 device=d), golden["match_rand"])
    tl, tr = synth.translated_noise_pair(40, 20, 5, 7)
    gl, gr = port.lightness(tl), port.lightness(tr)
    out = stk.match_boundary_pixels(gl, gr, np.ones((20, 40), np.uint8), stk.MatchConfig(5, 8),
                                    device=d)
    eq(out, golden["match_trans"])
    assert (out[2:18, 7:38] == 5).all()
    tl, tr = synth.translated_noise_pair(48, 30, 4, 12)
    gl, gr = port.lightness(tl), port.lightness(tr)
    eq(stk.match_boundary_pixels(gl, gr, synth.random_mask(48, 30, 13, 35), stk.MatchConfig(9, 16),
                                 device=d), golden["match_w9"])
    img = synth.random_gray(12, 8, 11)
    out = stk.match_boundary_pixels(img, img, np.ones((8, 12), np.uint8), stk.MatchConfig(3, 6),
                                    device=d)
    eq(out, golden["match_edge"])
    assert (out[1:7, 1] == 0).all() and (out[:, 0] == -1).all()


@pytest.mark.parametrize("w,h,win,D,pct", [
    (300, 40, 3, 7, 40), (257, 31, 9, 16, 25), (500, 60, 15, 64, 20), (640, 48, 21, 128, 19),
    (700, 70, 31, 256, 15), (130, 50, 5, 0, 50), (200, 25, 1, 33, 30), (64, 64, 25, 40, 30),
    (9, 9, 9, 16, 100), (8, 40, 9, 4, 100)])
def test_match_random_vs_oracle(sad_dev, stk, port, synth, w, h, win, D, pct):
    l = synth.random_gray(w, h, w + 3 * h)
    r = np.roll(l, -min(D, 5), axis=1) ^ (synth.random_gray(w, h, w * h) & 3)  # near-shift + noise
    m = synth.random_mask(w, h, 7 * w + h, pct)
    eq(stk.match_boundary_pixels(l, r, m, stk.MatchConfig(win, D), device=sad_dev),
       port.match(l, r, m, win, D))


@pytest.mark.parametrize("win,D", [(9, 16), (15, 64), (21, 128), (31, 256)])
def test_match_ws_extremes(dev, stk, port, synth, win, D):
    """K5c at its four compiled windows on multi-strip, multi-band frames with
    0/255 pixels (largest possible window sums: the u16x2 partial sums must not
    overflow) and a dense mask, against the per-pixel list kernel and the oracle."""
    w, h = 700, 160
    rng = np.random.default_rng(win * 1000 + D)
    l = (rng.integers(0, 2, (h, w), dtype=np.uint8) * 255).astype(np.uint8)
    r = np.roll(l, -3, axis=1)
    r[rng.random((h, w)) < 0.3] ^= 255
    m = synth.random_mask(w, h, win + D, 60)
    dev.set_sad_kernel("ws")
    a = stk.match_boundary_pixels(l, r, m, stk.MatchConfig(win, D), device=dev)
    dev.set_sad_kernel("list")
    b = stk.match_boundary_pixels(l, r, m, stk.MatchConfig(win, D), device=dev)
    dev.set_sad_kernel("auto")
    eq(a, b)
    eq(a, port.match(l, r, m, win, D))
    full = np.full((60, 400), 255, np.uint8)
    zero = np.zeros((60, 400), np.uint8)
    dev.set_sad_kernel("ws")
    out = stk.match_boundary_pixels(full, zero, np.ones((60, 400), np.uint8), stk.MatchConfig(win, D),
                                    device=dev)
    dev.set_sad_kernel("auto")
    eq(out, port.match(full, zero, np.ones((60, 400), np.uint8), win, D))


def test_match_ties_pick_smallest_d(sad_dev, stk, port):
    """Flat images: every candidate costs 0, the winner must be d = 0."""
    img = np.full((40, 200), 77, np.uint8)
    m = np.ones((40, 200), np.uint8)
    out = stk.match_boundary_pixels(img, img, m, stk.MatchConfig(9, 50), device=sad_dev)
    eq(out, port.match(img, img, m, 9, 50))
    assert set(np.unique(out)) <= {-1, 0}


def test_sad_cost(dev, stk, port, synth):
    l, r = synth.random_gray(16, 16, 3), synth.random_gray(16, 16, 4)
    for y in range(1, 15, 3):
        for x in range(1, 15, 2):
            for d in range(0, min(6, x - 1) + 1):
                assert stk.sad_cost(l, r, x, y, d, 3, device=dev) == port.sad_cost(l, r, x, y, d, 3)


def test_match_validation(dev, stk):
    a, b = np.zeros((8, 16), np.uint8), np.zeros((8, 12), np.uint8)
    with pytest.raises(stk.ParamError) as e:
        stk.match_boundary_pixels(a, b, np.ones((8, 16), np.uint8), device=dev)
    assert "16x8" in str(e.value) and "12x8" in str(e.value)
    with pytest.raises(stk.ParamError):
        stk.match_boundary_pixels(a, a, np.ones((4, 4), np.uint8), device=dev)
    for win, D in ((4, 16), (-3, 16), (3, -1)):
        with pytest.raises(stk.ParamError):
            stk.match_boundary_pixels(a, a, np.ones((8, 16), np.uint8), stk.MatchConfig(win, D),
                                      device=dev)


# -------------------------------------------------------------- K6 / K7 -----
def test_reconstruct_golden(dev, stk, golden):
    for s, f, p0, p1 in zip(golden["rec_sparse"], golden["rec_fill"], golden["rec_peek0"],
                            golden["rec_peek1"]):
        eq(stk.fill_scanlines(s, device=dev), f)
        eq(stk.peek_columns(f, 0, device=dev), p0)
        eq(stk.peek_columns(f, 1, device=dev), p1)


def test_reconstruct_known_answers(dev, stk):
    U = -1

    def row(v):
        return stk.fill_scanlines(np.array([v], np.int16), device=dev)[0].tolist()

    def col(v, t):
        return stk.peek_columns(np.array(v, np.int16)[:, None], t, device=dev)[:, 0].tolist()

    assert row([5, U, U, 5]) == [5, 5, 5, 5]
    assert row([5, U, U, 7]) == [5, U, U, 7]
    assert row([3, U, 3, U, 9]) == [3, 3, 3, U, 9]
    assert row([U, U, 2, U, 2, U]) == [U, U, 2, 2, 2, U]
    assert col([4, U, 10], 1) == [4, 4, 10]
    assert col([6, U, 7], 1) == [6, 6, 7]
    assert col([6, U, 6], 0) == [6, 6, 6]
    assert col([U, 3, 7], 1) == [3, 3, 7]
    assert col([U, 3, 7], 4) == [5, 3, 7]
    assert col([3, 7, U], 4) == [3, 7, 5]
    assert col([U, 3, U, U], 1) == [3, 3, 3, 3]
    assert col([U, U, U], 1) == [U, U, U]
    with pytest.raises(stk.ParamError):
        stk.peek_columns(np.zeros((4, 4), np.int16), -1, device=dev)


@pytest.mark.parametrize("w,h,pct", [(64, 1, 20), (1, 48, 20), (4096, 17, 3), (7, 2500, 2),
                                     (1000, 300, 19), (333, 333, 0), (50, 50, 100)])
def test_reconstruct_random_vs_oracle(dev, stk, port, synth, w, h, pct):
    s = synth.random_sparse(w, h, w ^ (h << 4), pct, 40)
    f = stk.fill_scanlines(s, device=dev)
    eq(f, port.fill_scanlines(s))
    for thr in (0, 1, 5):
        eq(stk.peek_columns(f, thr, device=dev), port.peek_columns(f, thr))


@pytest.mark.parametrize("w,h,p,vmax", [(320, 240, 0.3, 257), (64, 2304, 0.3, 257), (64, 4320, 0.02, 257),
                                        (66, 700, 0.05, 1024), (48, 300, 0.2, 32767), (2, 4321, 0.01, 32767)])
def test_peek_wide_values_vs_oracle(dev, stk, port, w, h, p, vmax):
    """K7 keeps both columns of a thread in int16x2 lanes (sign masks by PRMT,
    selects by LOP3): disparities with a high byte (>= 256, up to 32767), tall
    columns (many segments, load batches), thresholds up to beyond the int16
    range -- against the oracle's scalar int arithmetic."""
    rng = np.random.default_rng(w * 7919 + h)
    m = np.where(rng.random((h, w)) < p, rng.integers(0, vmax + 1, (h, w)), -1).astype(np.int16)
    for thr in (0, 1, 300, 40000):
        eq(stk.peek_columns(m, thr, device=dev), port.peek_columns(m, thr))


@pytest.mark.parametrize("w,h,p,vmax", [(256, 33, 0.2, 257), (4096, 7, 0.05, 32767), (64, 2, 0.5, 1024),
                                        (16, 1, 0.3, 300), (1024, 300, 0.02, 32767)])
def test_fill_wide_values_vs_oracle(dev, stk, port, w, h, p, vmax):
    """K6 v2 keeps two rows in int16x2 lanes (widths a multiple of 16): values
    with a high byte, odd heights (a lone last row), single rows."""
    rng = np.random.default_rng(w * 31 + h)
    m = np.where(rng.random((h, w)) < p, rng.integers(0, vmax + 1, (h, w)), -1).astype(np.int16)
    # runs of equal knowns so that gaps get filled
    m[:, ::7] = np.where(m[:, ::7] >= 0, 5, m[:, ::7])
    eq(stk.fill_scanlines(m, device=dev), port.fill_scanlines(m))


# ----------------------------------------------------------------- K8 -------
def test_blur_map(dev, stk, golden, port, synth):
    eq(stk.build_blur_map(np.array([[2, 4, 11, 7]], np.int16), [(3, 5), (10, 12)], 16, device=dev),
       golden["bm_simple"])
    assert stk.build_blur_map(np.array([[5, -1, 5]], np.int16), [(0, 16)], 16,
                              device=dev).tolist() == [[0, 1, 0]]
    for rng in ([], [(5, 3)], [(-1, 3)], [(3, 17)]):
        with pytest.raises(stk.ParamError):
            stk.build_blur_map(np.zeros((2, 2), np.int16), rng, 16, device=dev)
    d = synth.random_sparse(77, 31, 900, 80, 12)
    eq(stk.build_blur_map(d, [(2, 4), (7, 7)], 12, device=dev), port.blur_map(d, [(2, 4), (7, 7)], 12))


@pytest.mark.parametrize("exact", [False, True])
def test_selective_blur(dev, stk, golden, port, synth, exact):
    tol = 0 if exact else BLUR_TOL_LSB
    k9 = stk.gaussian_kernel(2.0, 9)
    img, msk = synth.random_rgb(33, 27, 45), synth.random_mask(33, 27, 46, 40)
    out = stk.selective_blur(img, msk, k9, sigma=2.0, exact=exact, device=dev)
    assert np.abs(out.astype(int) - golden["blur_rand"].astype(int)).max() <= tol
    img, msk = synth.random_rgb(21, 15, 43), synth.random_mask(21, 15, 44, 50)
    out = stk.selective_blur(img, msk, k9, sigma=2.0, exact=exact, device=dev)
    assert (out[msk == 0] == img[msk == 0]).all()  # sharp pixels keep their bytes
    assert np.abs(out.astype(int) - golden["blur_sharp_next"].astype(int)).max() <= tol
    edge = np.zeros((3, 3, 3), np.uint8)
    edge[0, 0] = 255
    out = stk.selective_blur(edge, np.ones((3, 3), np.uint8), stk.gaussian_kernel(1.0, 3), sigma=1.0,
                             exact=exact, device=dev)
    assert np.abs(out.astype(int) - golden["blur_edge"].astype(int)).max() <= tol
    # identities (test_refocus.cpp:125-160)
    img = synth.random_rgb(17, 13, 40)
    assert (stk.selective_blur(img, np.zeros((13, 17), np.uint8), stk.gaussian_kernel(2.0, 13),
                               sigma=2.0, exact=exact, device=dev) == img).all()
    img = synth.random_rgb(9, 9, 41)
    assert (stk.selective_blur(img, np.ones((9, 9), np.uint8), stk.gaussian_kernel(1.0, 1),
                               sigma=1.0, exact=exact, device=dev) == img).all()
    const = np.zeros((7, 11, 3), np.uint8)
    const[..., 0], const[..., 1:] = 90, 140
    assert (stk.selective_blur(const, synth.random_mask(11, 7, 42, 50), stk.gaussian_kernel(1.5, 9),
                               sigma=1.5, exact=exact, device=dev) == const).all()


@pytest.mark.parametrize("sigma,size,w,h", [(0.5, 5, 640, 480), (2.0, 13, 640, 480),
                                            (8.0, 49, 320, 240), (3.0, 0, 101, 57)])
def test_selective_blur_vs_oracle(dev, stk, port, synth, sigma, size, w, h):
    size = size or stk.default_kernel_size(sigma)
    img = synth.random_rgb(w, h, w + h)
    msk = synth.random_mask(w, h, w * h, 70)
    want = port.selective_blur(img, msk, sigma, size)
    fast = stk.selective_blur(img, msk, stk.gaussian_kernel(sigma, size), sigma=sigma, device=dev)
    assert np.abs(fast.astype(int) - want.astype(int)).max() <= BLUR_TOL_LSB
    exact = stk.selective_blur(img, msk, stk.gaussian_kernel(sigma, size), sigma=sigma, exact=True,
                               device=dev)
    eq(exact, want)
