"""Small workload for compute-sanitizer: one refocus frame per SAD kernel at
a ragged size, the stage entries (B1 stage modes, run-CCL labels / prune,
matching, the wide-parameter kernels) and a wide-blur frame."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2001_07809_b200 import stereotk as stk, synth

dev = stk.Device(0, slots=2)
l, r = synth.dead_leaves(333, 211, 24, frame=1)
for k in ("ws", "strip", "list", "auto"):
    dev.set_sad_kernel(k)
    stk.run_refocus_pipeline(l, r, stk.PipelineConfig(k=5, window=9, max_disparity=24),
                             stk.FocusSpec([(8, 24)], 2.0), device=dev)
dev.set_sad_kernel("auto")
stk.run_refocus_pipeline(l, r, stk.PipelineConfig(k=5, window=21, max_disparity=24),
                         stk.FocusSpec([(8, 24)], 8.0), device=dev)       # 49-tap v3
stk.run_refocus_pipeline(l, r, stk.PipelineConfig(k=5, window=65, max_disparity=40),
                         stk.FocusSpec([(8, 24)], 20.0), kernel_size=121, device=dev)  # wide SAD + global blur
g = stk.rgb_to_lightness(l, device=dev)
lab = (synth.random_gray(333, 211, 3).astype(np.uint16) * 7) % 300
stk.detect_boundaries(lab, device=dev)
m = synth.random_mask(333, 211, 4, 45)
stk.morph_fill(m, device=dev); stk.morph_remove(m, device=dev)
stk.label_components(m, device=dev); stk.prune_components(m, 0.04, device=dev)
stk.match_boundary_pixels(g, g, m, stk.MatchConfig(window=9, max_disparity=30), device=dev)
dev.close()
print("sanitize workload ok")
