"""Convert-stage time (CUDA events, StageTimes.convert) on 4K grey dead-leaves
frames and on 4K uniformly random RGB frames (the L* table's worst case)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2001_07809_b200 import stereotk as stk, synth

W, H = 4096, 2304
dev = stk.Device(0, W, H, slots=1)
cfg = stk.PipelineConfig(k=8, window=21, max_disparity=128)
focus = stk.FocusSpec([(64, 128)], 2.0)
rng = np.random.default_rng(5)
cases = {"grey dead-leaves": synth.dead_leaves(W, H, 128, frame=0),
         "random RGB": (rng.integers(0, 256, (H, W, 3), dtype=np.uint8),
                        rng.integers(0, 256, (H, W, 3), dtype=np.uint8))}
for name, (l, r) in cases.items():
    ts = []
    for i in range(6):
        t = stk.StageTimes()
        stk.run_depth_pipeline(l, r, cfg, t, full=False, device=dev)
        ts.append(t.convert)
    print(f"LUT={os.environ.get('STK_LSTAR_LUT', '1')} {name:18s} convert ms {np.median(ts[1:]):.4f}")
