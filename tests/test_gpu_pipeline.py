"""GPU parity of the whole frame (run_depth_pipeline / run_refocus_pipeline
through the C-ABI): every DepthResult intermediate bit-exact against the
compiled reference's golden frames and the oracle, the refocused image within
1 LSB (bit-exact in exact-blur mode), plus size-independent properties at the
benchmark's full 4096x2304 size, determinism and the async frame slots."""
import ctypes as C
import os

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BLUR_TOL_LSB = 1
INTERMEDIATES = ("left_lightness", "right_lightness", "labels", "boundary_raw", "boundary_refined",
                 "boundary_anchored", "sparse", "row_filled", "dense")


def eq(a, b, what=""):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    bad = int((a != b).sum())
    assert bad == 0, f"{what}: {bad} mismatching elements"


def run(stk, dev, l, r, k=10, window=9, D=16, thr=1, prune=0.04, focus=None, sigma=2.0,
        exact=False):
    cfg = stk.PipelineConfig(k=k, window=window, max_disparity=D, threshold=thr,
                             prune_fraction=prune)
    if focus is None:
        return stk.run_depth_pipeline(l, r, cfg, device=dev), None
    out = []
    img = stk.run_refocus_pipeline(l, r, cfg, stk.FocusSpec(focus, sigma, exact), depth_out=out,
                                   device=dev)
    return out[0], img


def check_golden(golden, tag, res, img, exact=False):
    for k in INTERMEDIATES:
        key = f"{tag}_{k}"
        if key in golden.files:
            eq(getattr(res, k), golden[key], key)
    st = golden[f"{tag}_stats"]
    assert [res.stats.pixels, res.stats.boundary_raw, res.stats.boundary_refined,
            res.stats.matched] == st.tolist()
    kit = golden[f"{tag}_kit"]
    assert res.clustering.k() == kit[0] and res.clustering.iterations_run == kit[1]
    assert (res.clustering.centers == golden[f"{tag}_centers"][: kit[0]]).all()
    key = f"{tag}_refocused"
    if img is not None and key in golden.files:
        d = np.abs(img.astype(int) - golden[key].astype(int)).max()
        assert d <= (0 if exact else BLUR_TOL_LSB), d


def test_pipeline_rectangle_scene_golden(dev, stk, golden, synth):
    l, r = synth.rectangle_scene_pair(96, 72, 4, 63)
    res, img = run(stk, dev, l, r, k=2, D=8, focus=[(3, 8)])
    check_golden(golden, "pipe_rect", res, img)
    res, img = run(stk, dev, l, r, k=2, D=8, focus=[(3, 8)], exact=True)
    check_golden(golden, "pipe_rect", res, img, exact=True)


def test_pipeline_self_match_golden(dev, stk, golden, synth):
    l, _ = synth.rectangle_scene_pair(96, 72, 0, 60)
    res, _ = run(stk, dev, l, l, k=2, D=8)
    check_golden(golden, "pipe_self", res, None)
    assert set(np.unique(res.sparse)) <= {-1, 0} and set(np.unique(res.dense)) <= {-1, 0}
    assert res.stats.matched > 0


@pytest.mark.parametrize("i", range(20))
def test_pipeline_criterion5_golden(dev, stk, golden, synth, i):
    """acceptance_main.cpp:262-272: 20 translated-noise scenes, D=12, focus {2,6}."""
    l, r = synth.translated_noise_pair(128, 96, i % 9, 500 + i)
    res, img = run(stk, dev, l, r, k=10, D=12, focus=[(2, 6)], sigma=1.5)
    check_golden(golden, f"crit5_{i}", res, img)


@pytest.mark.parametrize("s", range(1, 9))
def test_pipeline_criterion8_translation_recovery(dev, stk, golden, synth, s):
    """acceptance_main.cpp:443-489: shifts 1..8 recovered exactly."""
    l, r = synth.rectangle_scene_pair(160, 120, s, 700 + s)
    res, _ = run(stk, dev, l, r, k=2, window=9, D=16)
    check_golden(golden, f"crit8_{s}", res, None)


@pytest.mark.parametrize("tag", ["g2A", "g1"])
def test_pipeline_bench_scenes_golden(dev, stk, golden, synth, tag):
    if tag == "g2A":
        l, r = synth.dead_leaves(450, 375, 16, frame=0)
        kw = dict(k=4, window=9, D=16, focus=[(8, 16)])
    else:
        l, r = synth.bench_frame(200, 150, 7)
        kw = dict(k=10, window=9, D=16, focus=[(8, 16)])
    res, img = run(stk, dev, l, r, **kw)
    check_golden(golden, tag, res, img)
    res, img = run(stk, dev, l, r, exact=True, **kw)
    check_golden(golden, tag, res, img, exact=True)


@pytest.mark.parametrize("W,H,D,win,K,frame", [(1920, 1080, 64, 15, 6, 0), (640, 360, 40, 11, 5, 3),
                                               (301, 203, 20, 7, 3, 1), (128, 64, 31, 31, 8, 2)])
def test_pipeline_vs_oracle(dev, stk, port, synth, W, H, D, win, K, frame):
    l, r = synth.dead_leaves(W, H, D, frame=frame)
    focus = [(D // 2, D)]
    res, img = run(stk, dev, l, r, k=K, window=win, D=D, focus=focus)
    want = port.run_frame(l, r, k=K, window=win, max_disparity=D, focus=focus, sigma=2.0)
    for k in INTERMEDIATES:
        eq(getattr(res, k), want[k], k)
    assert np.abs(img.astype(int) - want["refocused"].astype(int)).max() <= BLUR_TOL_LSB
    assert res.stats.matched == want["stats"]["matched"]


def test_pipeline_4k_properties(dev, stk, port, synth):
    """Full benchmark size (4096x2304, D=128, w=21, K=8): the cheap stages are
    checked exactly against the oracle; SAD through list == strip kernels and
    an oracle spot check; structural invariants of the reconstruction."""
    W, H, D, win, K = 4096, 2304, 128, 21, 8
    l, r = synth.dead_leaves(W, H, D, frame=0)
    dev.set_sad_kernel("strip")
    a, img = run(stk, dev, l, r, k=K, window=win, D=D, focus=[(64, 128)])
    dev.set_sad_kernel("list")
    b, _ = run(stk, dev, l, r, k=K, window=win, D=D)
    dev.set_sad_kernel("ws")
    c_, _ = run(stk, dev, l, r, k=K, window=win, D=D)
    dev.set_sad_kernel("auto")
    eq(a.sparse, b.sparse, "strip vs list")
    eq(c_.sparse, b.sparse, "ws vs list")
    eq(a.left_lightness, port.lightness(l), "L*")
    eq(a.labels, a.clustering.bin_assignment[a.left_lightness], "labels")
    c, asg, it = port.kmeans(port.histogram(a.left_lightness), K)
    assert (a.clustering.centers == c).all() and a.clustering.iterations_run == it
    eq(a.boundary_raw, port.detect(a.labels), "detect")
    refined = port.prune(port.remove(port.fill(a.boundary_raw)), 0.04)
    eq(a.boundary_refined, refined, "refine")
    eq(a.boundary_anchored, port.anchors(refined, win // 2), "anchors")
    eq(a.row_filled, port.fill_scanlines(a.sparse), "fill")
    eq(a.dense, port.peek_columns(a.row_filled, 1), "peek")
    # SAD spot check against the per-pixel oracle cost
    ys, xs = np.nonzero(a.sparse >= 0)
    assert len(ys) == a.stats.matched and 0.17 < a.stats.matched_fraction < 0.21
    pick = np.random.default_rng(0).choice(len(ys), 300, replace=False)
    for i in pick:
        y, x = int(ys[i]), int(xs[i])
        dl = min(D, x - win // 2)
        costs = [port.sad_cost(a.left_lightness, a.right_lightness, x, y, d, win)
                 for d in range(dl + 1)]
        assert int(np.argmin(costs)) == a.sparse[y, x]
    # known pixels are never modified; sharp pixels keep their bytes
    k = a.sparse >= 0
    assert (a.row_filled[k] == a.sparse[k]).all()
    k = a.row_filled >= 0
    assert (a.dense[k] == a.row_filled[k]).all()
    sharp = (a.dense >= 64) & (a.dense <= 128)
    assert (img[sharp] == l[sharp]).all()


def test_pipeline_determinism_and_modes(dev, stk, synth):
    l, r = synth.dead_leaves(640, 480, 32, frame=5)
    outs = []
    for graphs in (True, False, True):
        dev.set_use_graphs(graphs)
        res, img = run(stk, dev, l, r, k=6, window=11, D=32, focus=[(10, 20)])
        outs.append((res.dense.copy(), img.copy()))
    dev.set_use_graphs(True)
    for d, i in outs[1:]:
        eq(d, outs[0][0], "dense")
        eq(i, outs[0][1], "refocused")
    lean = stk.run_depth_pipeline(l, r, stk.PipelineConfig(k=6, window=11, max_disparity=32),
                                  full=False, device=dev)
    eq(lean.dense, outs[0][0], "lean mode")
    # lean frames do not preset sparse (the row fill masks with the matchable
    # bits): a lean frame after other frames left their disparities in the
    # slot's sparse plane still equals the full-mode result
    for other in (6, 7):
        l2, r2 = synth.dead_leaves(640, 480, 32, frame=other)
        cfg2 = stk.PipelineConfig(k=6, window=11, max_disparity=32)
        full2 = stk.run_depth_pipeline(l2, r2, cfg2, device=dev)
        stk.run_depth_pipeline(l2, r2, cfg2, full=False, device=dev)
        lean = stk.run_depth_pipeline(l, r, stk.PipelineConfig(k=6, window=11, max_disparity=32),
                                      full=False, device=dev)
        eq(lean.dense, outs[0][0], "lean mode after other frames")
        eq(stk.run_depth_pipeline(l2, r2, cfg2, full=False, device=dev).dense, full2.dense, "lean, other")


def test_pipeline_stage_times(dev, stk, synth):
    l, r = synth.dead_leaves(450, 375, 16, frame=1)
    t = stk.StageTimes()
    res = stk.run_depth_pipeline(l, r, stk.PipelineConfig(k=4), times=t, device=dev)
    assert t.total() > 0.0
    assert t.total() == pytest.approx(t.convert + t.segment + t.boundary + t.match + t.fill + t.peek)
    assert res.stats.pixels == 450 * 375


def test_pipeline_errors(dev, stk):
    with pytest.raises(stk.ParamError) as e:
        stk.run_depth_pipeline(np.zeros((48, 64, 3), np.uint8), np.zeros((48, 32, 3), np.uint8),
                               device=dev)
    assert "64x48" in str(e.value) and "32x48" in str(e.value)
    z = np.zeros((10, 10, 3), np.uint8)
    with pytest.raises(stk.ParamError, match="window"):
        stk.run_depth_pipeline(z, z, stk.PipelineConfig(window=4), device=dev)
    with pytest.raises(stk.ParamError, match="add_border_anchors"):
        stk.run_depth_pipeline(z, z, stk.PipelineConfig(window=11), device=dev)
    with pytest.raises(stk.ParamError, match="k must be at least 1, got 0"):
        e0 = np.zeros((0, 0, 3), np.uint8)
        stk.run_depth_pipeline(e0, e0, device=dev)
    with pytest.raises(stk.ParamError, match="bad focus range"):
        stk.run_refocus_pipeline(z, z, stk.PipelineConfig(window=3), stk.FocusSpec([(3, 17)]),
                                 device=dev)


def test_async_slots_match_sync(dev, stk, synth):
    """Three frames in flight on three slots (pinned host buffers) give the same
    bytes as synchronous frames."""
    from paper_2001_07809_b200 import _lib

    L = _lib.lib()
    W, H = 512, 256
    cfg = stk.PipelineConfig(k=5, window=9, max_disparity=24)
    focus = stk.FocusSpec([(8, 24)], 2.0)
    frames = [synth.dead_leaves(W, H, 24, frame=i) for i in range(6)]
    want = [stk.run_refocus_pipeline(l, r, cfg, focus, device=dev) for l, r in frames]
    c_cfg = cfg.c()
    c_focus, _keep = stk._focus_c(focus, 0)
    outs = [np.empty((H, W, 3), np.uint8) for _ in frames]
    fo = [_lib.StkFrameOut() for _ in frames]
    for i in range(len(frames)):
        fo[i].refocused = outs[i].ctypes.data
    pending = [None] * 3
    for i, (l, r) in enumerate(frames):
        s = i % 3
        if pending[s] is not None:
            stk._raise(L.stk_frame_wait(dev.h, s, None, None, None), dev.h)
        stk._raise(L.stk_frame_submit(dev.h, s, l.ctypes.data, r.ctypes.data, W, H, C.byref(c_cfg),
                                      C.byref(c_focus), C.byref(fo[i]), 0), dev.h)
        pending[s] = i
    for s in range(3):
        stk._raise(L.stk_frame_wait(dev.h, s, None, None, None), dev.h)
    for a, b in zip(outs, want):
        eq(a, b, "async")


def test_frame_lightness_all_2pow24_triples(dev, stk, port):
    """The frame path's K1 (both views in one launch, bucket words + exact tie
    reads) on every RGB triple, left and right, against the pinned oracle."""
    v = np.arange(256, dtype=np.uint8)
    rgb = np.stack(np.meshgrid(v, v, v, indexing="ij"), -1).reshape(4096, 4096, 3)
    rgb_r = np.ascontiguousarray(rgb[::-1])
    res, _ = run(stk, dev, rgb, rgb_r, k=4, window=9, D=8)
    want = port.lightness(rgb)
    eq(res.left_lightness, want, "left_lightness")
    eq(res.right_lightness, want[::-1], "right_lightness")


def test_pipeline_8k_config_e(dev, stk, synth, port):
    """Config E (7680x4320, D=256, w=31, K=8, sigma=8 -> 49-tap blur): the
    warp-specialised SAD (G=5 lanes per column group for w=31) equals the
    list kernel on every pixel; every O(N) stage equals the oracle exactly on
    the GPU's own inputs (L*, fused histogram -> K-Means, detect, refine,
    anchors, fill, peek); reconstruction and blur invariants hold."""
    W, H, D, win, K = 7680, 4320, 256, 31, 8
    l, r = synth.dead_leaves(W, H, D, frame=0)
    dev.set_sad_kernel("ws")
    a, img = run(stk, dev, l, r, k=K, window=win, D=D, focus=[(128, 256)], sigma=8.0)
    dev.set_sad_kernel("list")
    b, _ = run(stk, dev, l, r, k=K, window=win, D=D)
    dev.set_sad_kernel("auto")
    eq(a.sparse, b.sparse, "ws vs list")
    assert 0.1 < a.stats.matched_fraction < 0.3
    eq(a.left_lightness, port.lightness(l), "L* (8K)")
    c, _, it = port.kmeans(port.histogram(a.left_lightness), K)
    assert (a.clustering.centers == c).all() and a.clustering.iterations_run == it
    eq(a.boundary_raw, port.detect(a.labels), "detect (8K)")
    refined = port.prune(port.remove(port.fill(a.boundary_raw)), 0.04)
    eq(a.boundary_refined, refined, "refine (8K)")
    eq(a.boundary_anchored, port.anchors(refined, win // 2), "anchors (8K)")
    eq(a.row_filled, port.fill_scanlines(a.sparse), "fill (8K)")
    eq(a.dense, port.peek_columns(a.row_filled, 1), "peek (8K)")
    k = a.sparse >= 0
    assert (a.row_filled[k] == a.sparse[k]).all()
    k = a.row_filled >= 0
    assert (a.dense[k] == a.row_filled[k]).all()
    sharp = (a.dense >= 128) & (a.dense <= 256)
    assert (img[sharp] == l[sharp]).all()
    assert (img[~sharp] != l[~sharp]).any()


def test_frame_lightness_lut_option_all_2pow24_triples(tmp_path, port):
    """The opt-in exact L* table (STK_LSTAR_LUT=1, read once per process, so a
    subprocess): every RGB triple through the frame path, both views, equals
    the pinned oracle."""
    import subprocess
    import sys

    v = np.arange(256, dtype=np.uint8)
    rgb = np.stack(np.meshgrid(v, v, v, indexing="ij"), -1).reshape(4096, 4096, 3)
    np.save(tmp_path / "rgb.npy", rgb)
    code = f"""
import sys, numpy as np
sys.path.insert(0, {ROOT!r})
from paper_2001_07809_b200 import stereotk as stk
rgb = np.load({str(tmp_path / 'rgb.npy')!r})
res = stk.run_depth_pipeline(rgb, np.ascontiguousarray(rgb[::-1]),
                             stk.PipelineConfig(k=4, window=9, max_disparity=8))
np.save({str(tmp_path / 'l.npy')!r}, res.left_lightness)
np.save({str(tmp_path / 'r.npy')!r}, res.right_lightness)
"""
    env = dict(os.environ, STK_LSTAR_LUT="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    want = port.lightness(rgb)
    eq(np.load(tmp_path / "l.npy"), want, "lut left_lightness")
    eq(np.load(tmp_path / "r.npy"), want[::-1], "lut right_lightness")


@pytest.mark.parametrize("sigma", [3.0, 5.0, 8.0])
def test_pipeline_wide_blur_vs_oracle(dev, stk, port, synth, sigma):
    """Wide kernels (sigma 3 / 5 / 8 -> 19 / 31 / 49 taps; 8 is config E's
    blur) through the frame path's separable blur, against the oracle's FP64
    2-D blur: <= 1 LSB."""
    l, r = synth.dead_leaves(320, 240, 16, frame=4)
    res, img = run(stk, dev, l, r, k=4, window=9, D=16, focus=[(8, 16)], sigma=sigma)
    want = port.run_frame(l, r, k=4, window=9, max_disparity=16, focus=[(8, 16)], sigma=sigma)
    eq(res.dense, want["dense"], "dense")
    assert np.abs(img.astype(int) - want["refocused"].astype(int)).max() <= BLUR_TOL_LSB


# sigma -> kernel size 2 ceil(3 sigma) + 1: 3, 5, 7, 9, 11, (13: default), 15, 17, and the
# wide tensor-core tiles 19 (3.0), 25, 31, 37, 43, 49 (8.0: config E)
@pytest.mark.parametrize("sigma", [0.3, 0.6, 1.0, 1.3, 1.6, 2.3, 2.6, 3.0, 4.0, 5.0, 6.0, 7.0, 8.0])
def test_pipeline_tc_blur_sizes_vs_oracle(dev, stk, port, synth, sigma):
    """Every kernel size of the tensor-core blur (K8t, K <= 17 and 19..49) through the
    frame path against the oracle's FP64 2-D blur: <= 1 LSB everywhere and
    almost everywhere exact (hi/lo f16 splits carry ~22 bits, so only sums
    within ~1e-4 of a rounding boundary may differ)."""
    l, r = synth.dead_leaves(320, 240, 16, frame=5)
    res, img = run(stk, dev, l, r, k=4, window=9, D=16, focus=[(8, 16)], sigma=sigma)
    want = port.run_frame(l, r, k=4, window=9, max_disparity=16, focus=[(8, 16)], sigma=sigma)
    eq(res.dense, want["dense"], "dense")
    d = np.abs(img.astype(int) - want["refocused"].astype(int))
    assert d.max() <= BLUR_TOL_LSB
    assert (d != 0).mean() < 1e-3, (d != 0).mean()


@pytest.mark.parametrize("W,H,sigma", [(333, 201, 2.0), (100, 50, 2.6), (7, 5, 1.0), (136, 33, 2.0),
                                       (264, 64, 0.6), (130, 31, 2.3), (333, 201, 8.0), (150, 90, 3.0),
                                       (7, 5, 5.0), (176, 40, 6.0)])
def test_pipeline_tc_blur_edge_shapes(dev, stk, port, synth, W, H, sigma):
    """K8t at shapes that exercise its slow paths: W not a multiple of 4
    (unaligned rows), W < 136 (no CTA has its staged columns inside the
    image), partial tiles in x and y, a frame smaller than one tile."""
    D = 8
    l, r = synth.dead_leaves(W, H, D, frame=3)
    res, img = run(stk, dev, l, r, k=3, window=3, D=D, focus=[(2, 6)], sigma=sigma)
    want = port.run_frame(l, r, k=3, window=3, max_disparity=D, focus=[(2, 6)], sigma=sigma)
    eq(res.dense, want["dense"], "dense")
    assert np.abs(img.astype(int) - want["refocused"].astype(int)).max() <= BLUR_TOL_LSB


def test_graph_survives_focus_table_reallocation(dev, stk, port, synth):
    """A stage entry that grows the slot's focus tables (a 67x67 blur kernel:
    > 4096 weights; max_disparity >= 1024: > 1024 LUT entries) between two
    graph-replayed frames of the same geometry must not leave the frame graph
    reading freed tables (stk_capi.cu upload_focus)."""
    W, H = 320, 240
    l, r = synth.dead_leaves(W, H, 16, frame=2)
    want = port.run_frame(l, r, k=4, window=9, max_disparity=16, focus=[(8, 16)], sigma=2.0)
    res, img = run(stk, dev, l, r, k=4, window=9, D=16, focus=[(8, 16)])
    assert np.abs(img.astype(int) - want["refocused"].astype(int)).max() <= BLUR_TOL_LSB
    # grow the weights (67 x 67 taps) and the LUT (D = 1100) on the same slot
    bmap = np.ones((H, W), np.uint8)
    stk.selective_blur(l, bmap, stk.gaussian_kernel(11.0, 67), sigma=11.0, device=dev)
    stk.build_blur_map(np.zeros((H, W), np.int16), [(0, 5)], 1100, device=dev)
    res2, img2 = run(stk, dev, l, r, k=4, window=9, D=16, focus=[(8, 16)])
    eq(res2.dense, want["dense"], "dense after realloc")
    eq(img2, img, "refocused after realloc")


def test_wide_blur_tile_edge_shape(dev, stk, ref, synth):
    """K = 49 (sigma 8) at W = 32 (mod 128), H = h (mod 16): the v3 interior
    fast path's last staged row ends exactly at the buffer end (ADVICE r1:
    k_blur.cu interior guard)."""
    W, H = 1440, 1080
    l, r = synth.dead_leaves(W, H, 32, frame=6)
    res, img = run(stk, dev, l, r, k=5, window=11, D=32, focus=[(16, 32)], sigma=8.0)
    want = ref.run_frame(l, r, k=5, window=11, max_disparity=32, focus=[(16, 32)], sigma=8.0,
                         workers=os.cpu_count() or 1)
    for k in INTERMEDIATES:
        eq(getattr(res, k), want[k], k)
    assert np.abs(img.astype(int) - want["refocused"].astype(int)).max() <= BLUR_TOL_LSB



def test_async_slots_focus_changes_per_frame(dev, stk, synth):
    """A video whose focus ranges and sigma change every frame: frames in
    flight on three slots (focus tables uploaded stream-ordered, no host
    synchronisation) give the same bytes as synchronous frames, and every
    frame after the first per slot replays the slot's CUDA graph (same kernel
    size: no re-capture)."""
    from paper_2001_07809_b200 import _lib

    L = _lib.lib()
    W, H = 512, 256
    cfg = stk.PipelineConfig(k=5, window=9, max_disparity=24)
    frames = [synth.dead_leaves(W, H, 24, frame=i) for i in range(9)]
    focuses = [stk.FocusSpec([(i % 5, 10 + i)], 1.5 + 0.05 * (i % 3)) for i in range(9)]  # 11 taps
    want = [stk.run_refocus_pipeline(l, r, cfg, fo, device=dev) for (l, r), fo in zip(frames, focuses)]
    c_cfg = cfg.c()
    keep = []
    outs = [np.empty((H, W, 3), np.uint8) for _ in frames]
    fo_c = [_lib.StkFrameOut() for _ in frames]
    info = _lib.StkFrameInfo()
    graphs = []
    pending = [None] * 3
    for i, (l, r) in enumerate(frames):
        s = i % 3
        if pending[s] is not None:
            stk._raise(L.stk_frame_wait(dev.h, s, None, None, C.byref(info)), dev.h)
            graphs.append((pending[s], info.graph, info.captured))
        fo_c[i].refocused = outs[i].ctypes.data
        c_focus, k = stk._focus_c(focuses[i], 0)
        keep.append((c_focus, k))
        stk._raise(L.stk_frame_submit(dev.h, s, l.ctypes.data, r.ctypes.data, W, H, C.byref(c_cfg),
                                      C.byref(c_focus), C.byref(fo_c[i]), 0), dev.h)
        pending[s] = i
    for s in range(3):
        stk._raise(L.stk_frame_wait(dev.h, s, None, None, C.byref(info)), dev.h)
        graphs.append((pending[s], info.graph, info.captured))
    for a, b in zip(outs, want):
        eq(a, b, "async focus change")
    assert all(g == 1 for _, g, _ in graphs)
    # slots 1 and 2 capture on their first frame; every later frame replays
    # (slot 0 already holds the synchronous frames' graph of this geometry)
    assert [i for i, _, cap in graphs if cap] == [1, 2], graphs


def test_4k_frames_deterministic_across_slots(dev, stk, synth):
    """Twelve 4K frames (two distinct pairs) through three async slots with
    graphs: every repeat of a pair gives byte-identical dense disparity and
    refocused image (the union-find phases run lock-free, in any order)."""
    from paper_2001_07809_b200 import _lib

    L = _lib.lib()
    W, H, D = 4096, 2304, 128
    cfg = stk.PipelineConfig(k=8, window=21, max_disparity=D)
    c_cfg = cfg.c()
    c_focus, _keep = stk._focus_c(stk.FocusSpec([(64, 128)], 2.0), 0)
    pairs = [synth.dead_leaves(W, H, D, frame=i) for i in (3, 4)]
    n = 12
    outs = [(np.empty((H, W, 3), np.uint8), np.empty((H, W), np.int16)) for _ in range(n)]
    fo = [_lib.StkFrameOut() for _ in range(n)]
    pending = [None] * 3
    for i in range(n):
        s = i % 3
        if pending[s] is not None:
            stk._raise(L.stk_frame_wait(dev.h, s, None, None, None), dev.h)
        fo[i].refocused = outs[i][0].ctypes.data
        fo[i].dense = outs[i][1].ctypes.data
        l, r = pairs[i % 2]
        stk._raise(L.stk_frame_submit(dev.h, s, l.ctypes.data, r.ctypes.data, W, H, C.byref(c_cfg),
                                      C.byref(c_focus), C.byref(fo[i]), 0), dev.h)
        pending[s] = i
    for s in range(3):
        stk._raise(L.stk_frame_wait(dev.h, s, None, None, None), dev.h)
    for i in range(2, n):
        eq(outs[i][1], outs[i % 2][1], f"dense repeat {i}")
        eq(outs[i][0], outs[i % 2][0], f"refocused repeat {i}")


@pytest.mark.parametrize("case", ["uniform", "two_levels", "thin_row", "thin_col", "tiny", "window1"])
def test_pipeline_degenerate_frames_vs_oracle(dev, stk, port, synth, case):
    """Frames at the edges of the algorithm: a uniform frame (one occupied
    bin, no boundary, everything unknown -> everything blurred), two grey
    levels with K = 8 (k = min(K, occupied) = 2), single-row / single-column
    frames, a 3x3 frame and window 1: every intermediate and the refocused
    image against the oracle."""
    rng = np.random.default_rng(11)
    k, win, D, focus = 8, 9, 16, [(4, 12)]
    if case == "uniform":
        l = np.full((240, 320, 3), 97, np.uint8)
        r = l.copy()
    elif case == "two_levels":
        l = np.where(rng.random((200, 300, 1)) < 0.5, 40, 200).astype(np.uint8).repeat(3, axis=2)
        r = np.roll(l, -3, axis=1)
    elif case == "thin_row":
        l, r = synth.dead_leaves(4096, 1, 16, frame=1)
        win = 1
    elif case == "thin_col":
        l, r = synth.dead_leaves(1, 2048, 16, frame=2)
        win = 1
    elif case == "tiny":
        l, r = synth.dead_leaves(3, 3, 2, frame=3)
        win, D, focus = 3, 2, [(0, 1)]
    else:
        l, r = synth.dead_leaves(257, 129, 16, frame=4)
        win = 1
    res, img = run(stk, dev, l, r, k=k, window=win, D=D, focus=focus)
    want = port.run_frame(l, r, k=k, window=win, max_disparity=D, focus=focus, sigma=2.0)
    for name in INTERMEDIATES:
        eq(getattr(res, name), want[name], f"{case} {name}")
    assert np.abs(img.astype(int) - want["refocused"].astype(int)).max() <= BLUR_TOL_LSB
    assert res.stats.matched == want["stats"]["matched"]
