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


@pytest.mark.parametrize("cap", [None, "0"])
def test_dot_grid_frame_many_components(cap):
    """A dot-grid frame (a dark dot every 4 px on a grey field, a few bright
    lines, +-2 noise): each dot leaves a boundary ring, 45.9 K region roots --
    beyond B3b's shared-memory forest, so B3 unites on the global forest (with
    STK_UNITE_CAP=0 every call of the process does).  The whole DepthResult
    bit-exact, the refocused image <= 1 LSB, in a fresh process per setting."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2001_07809_b200 import stereotk as stk
import oracle
port = oracle.port()
rng = np.random.default_rng(5)
W, H, D = 1024, 768, 16
l = np.full((H, W, 3), 128, np.uint8)
l[2::4, 2::4] = 0
l[::97, :] = 255
l = (l.astype(int) + rng.integers(0, 3, l.shape)).clip(0, 255).astype(np.uint8)
r = np.roll(l, -5, axis=1)
d = stk.Device(0, slots=1)
cfg = stk.PipelineConfig(k=8, window=5, max_disparity=D)
out = []
img = stk.run_refocus_pipeline(l, r, cfg, stk.FocusSpec([(4, 9)], 1.0), depth_out=out, device=d)
want = port.run_frame(l, r, k=8, window=5, max_disparity=D, focus=[(4, 9)], sigma=1.0)
for key in %r:
    a = np.asarray(getattr(out[0], key))
    assert a.shape == want[key].shape and (a == want[key]).all(), key
assert np.abs(img.astype(int) - want["refocused"].astype(int)).max() <= 1
d.close()
print("ok")
""" % (KEYS,)
    env = dict(os.environ)
    if cap is not None:
        env["STK_UNITE_CAP"] = cap
    r = subprocess.run([sys.executable, "-c", code, root], capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]
