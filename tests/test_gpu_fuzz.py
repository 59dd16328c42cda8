"""Randomised whole frames (the frame path end to end) against the oracle:
random sizes, windows, disparity ranges, cluster counts, focus ranges and blur
sigmas -- every DepthResult intermediate bit-exact, the refocused image <= 1
LSB.  scripts/fuzz_frames.py runs the same sweep at scale (450 frames green at
the end of round 2)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KEYS = ("left_lightness", "right_lightness", "labels", "boundary_raw", "boundary_refined",
        "boundary_anchored", "sparse", "row_filled", "dense")


@pytest.mark.parametrize("case", range(24))
def test_random_frame_vs_oracle(dev, stk, port, synth, case):
    rng = np.random.default_rng(1000 + case)
    W = int(rng.integers(8, 600))
    H = int(rng.integers(8, 360))
    win = int(rng.choice([1, 3, 5, 9, 15, 21, 31]))
    D = int(rng.integers(1, min(W, 260)))
    k = int(rng.integers(2, 13))
    sigma = float(rng.choice([0.3, 0.6, 1.0, 1.6, 2.0, 2.6, 3.0, 5.0, 8.0]))
    lo = int(rng.integers(0, D))
    hi = int(rng.integers(lo + 1, D + 1))
    l, r = synth.dead_leaves(W, H, D, frame=case)
    cfg = stk.PipelineConfig(k=k, window=win, max_disparity=D)
    out = []
    img = stk.run_refocus_pipeline(l, r, cfg, stk.FocusSpec([(lo, hi)], sigma), depth_out=out, device=dev)
    want = port.run_frame(l, r, k=k, window=win, max_disparity=D, focus=[(lo, hi)], sigma=sigma)
    for key in KEYS:
        a = np.asarray(getattr(out[0], key))
        assert a.shape == want[key].shape and (a == want[key]).all(), (key, W, H, win, D, k, sigma)
    assert np.abs(img.astype(int) - want["refocused"].astype(int)).max() <= 1
