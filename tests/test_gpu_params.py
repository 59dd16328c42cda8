"""The reference's full parameter range on the GPU (stereo.cpp:49-57 accepts any
odd window >= 1 and any max_disparity >= 0; refocus.cpp:16-43 any odd kernel
size): windows beyond the fast SAD kernels (> 31 / > 63), disparity ranges
beyond the 10-bit argmin keys (> 1023), and blur kernels too wide for a
shared-memory tile, each against the compiled reference (all host cores)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

WORKERS = os.cpu_count() or 1


def _eq(a, b, what):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    bad = int((a != b).sum())
    assert bad == 0, f"{what}: {bad} mismatching elements"


@pytest.mark.parametrize("window,D", [(65, 1100), (101, 40), (3, 5000), (33, 1024), (63, 2047)])
def test_match_any_window_and_range(dev, stk, ref, synth, window, D):
    W, H = 1300, max(2 * window, 90)
    l, r = synth.dead_leaves(W, H, 200, frame=1)
    gl, gr = ref.lightness(l), ref.lightness(r)
    mask = synth.random_mask(W, H, window + D, 1)
    got = stk.match_boundary_pixels(gl, gr, mask, stk.MatchConfig(window=window, max_disparity=D),
                                    device=dev)
    want = ref.match(gl, gr, mask, window, D, workers=WORKERS)
    _eq(got, want, f"match w={window} D={D}")
    assert (got >= 0).sum() > 0


def test_pipeline_wide_window_and_range(dev, stk, ref, synth):
    """run_refocus_pipeline at window 65, max_disparity 1100 (the SAD's wide
    fallback) with a 121-tap blur (the global-memory fallback): every
    intermediate exact, refocused <= 1 LSB; exact mode bit-identical."""
    W, H, win, D = 1200, 96, 65, 1100
    l, r = synth.dead_leaves(W, H, 300, frame=2)
    cfg = stk.PipelineConfig(k=5, window=win, max_disparity=D)
    for exact in (False, True):
        out = []
        img = stk.run_refocus_pipeline(l, r, cfg, stk.FocusSpec([(0, 150)], 20.0, exact),
                                       kernel_size=121, depth_out=out, device=dev)
        want = ref.run_frame(l, r, k=5, window=win, max_disparity=D, focus=[(0, 150)], sigma=20.0,
                             kernel_size=121, workers=WORKERS)
        for name in ("left_lightness", "labels", "boundary_refined", "boundary_anchored", "sparse",
                     "row_filled", "dense"):
            _eq(getattr(out[0], name), want[name], name)
        d = np.abs(img.astype(int) - want["refocused"].astype(int)).max()
        assert d <= (0 if exact else 1), d


@pytest.mark.parametrize("size,exact", [(121, False), (121, True), (151, False), (151, True), (99, True)])
def test_selective_blur_wide_kernels(dev, stk, ref, synth, size, exact):
    l, _ = synth.dead_leaves(300, 200, 16, frame=3)
    bmap = synth.random_mask(300, 200, size, 50)
    sigma = size / 6.0
    got = stk.selective_blur(l, bmap, stk.gaussian_kernel(sigma, size), sigma=sigma, exact=exact,
                             device=dev)
    want = ref.selective_blur(l, bmap, sigma, size, workers=WORKERS)
    d = np.abs(got.astype(int) - want.astype(int)).max()
    assert d <= (0 if exact else 1), d
    assert (got[bmap == 0] == l[bmap == 0]).all()
