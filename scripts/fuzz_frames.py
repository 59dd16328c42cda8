"""Randomised whole-frame parity sweep (GPU vs the oracle port): random sizes,
disparity ranges, windows, cluster counts, focus ranges and blur sigmas.
Every DepthResult intermediate bit-exact, refocused <= 1 LSB.
  python scripts/fuzz_frames.py [n_cases] [seed]"""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2001_07809_b200 import stereotk as stk, synth
import oracle

KEYS = ("left_lightness", "right_lightness", "labels", "boundary_raw", "boundary_refined",
        "boundary_anchored", "sparse", "row_filled", "dense")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
port = oracle.port()
dev = stk.Device(0, 64, 64)
bad = 0
for i in range(n):
    W = int(rng.integers(8, 720)); H = int(rng.integers(8, 420))
    win = int(rng.choice([1, 3, 5, 9, 15, 21, 31]))
    D = int(rng.integers(0, min(W, 260)))
    k = int(rng.integers(2, 13))
    sigma = float(rng.choice([0.3, 0.6, 1.0, 1.6, 2.0, 2.6, 3.0, 5.0, 8.0]))
    lo = int(rng.integers(0, max(1, D))); hi = int(rng.integers(lo + 1, D + 2))
    focus = [(lo, hi)]
    l, r = synth.dead_leaves(W, H, max(D, 1), frame=i)
    cfg = stk.PipelineConfig(k=k, window=win, max_disparity=D)
    try:
        out = []
        img = stk.run_refocus_pipeline(l, r, cfg, stk.FocusSpec(focus, sigma), depth_out=out, device=dev)
        res = out[0]
    except stk.ParamError as e:
        print(f"case {i}: ParamError {e}")
        continue
    want = port.run_frame(l, r, k=k, window=win, max_disparity=D, focus=focus, sigma=sigma)
    msg = []
    for key in KEYS:
        a, b = np.asarray(getattr(res, key)), want[key]
        if a.shape != b.shape or (a != b).any():
            msg.append(f"{key}: {int((a != b).sum()) if a.shape == b.shape else 'shape'}")
    dmax = int(np.abs(img.astype(int) - want["refocused"].astype(int)).max())
    if dmax > 1:
        msg.append(f"refocused max diff {dmax}")
    status = "ok" if not msg else "MISMATCH " + "; ".join(msg)
    bad += bool(msg)
    print(f"case {i}: {W}x{H} w={win} D={D} k={k} sigma={sigma} focus={focus}: {status}", flush=True)
print(f"{n - bad}/{n} cases ok")
sys.exit(1 if bad else 0)
