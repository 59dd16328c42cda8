"""Run a few device-resident frames of a config (for ncu / nsys-free profiling)."""
import argparse, ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2001_07809_b200 import _lib, synth, stereotk as stk
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C")
ap.add_argument("--frames", type=int, default=3)
ap.add_argument("--sad", default="auto")
ap.add_argument("--graphs", type=int, default=0)
a = ap.parse_args()
W, H, D, win, K, focus, sigma = bench.CONFIGS[a.config]
dev = stk.Device(0, W, H, slots=1)
dev.set_sad_kernel(a.sad)
dev.set_use_graphs(bool(a.graphs))
l, r = synth.dead_leaves(W, H, D, frame=0)
dl, dr = torch.from_numpy(l).cuda(), torch.from_numpy(r).cuda()
o = torch.empty((H, W, 3), dtype=torch.uint8, device="cuda")
dd = torch.empty((H, W), dtype=torch.int16, device="cuda")
cfg = stk.PipelineConfig(k=K, window=win, max_disparity=D).c()
fc, keep = stk._focus_c(stk.FocusSpec(focus, sigma), 0)
L = _lib.lib()
for i in range(a.frames):
    stk._raise(L.stk_frame_submit_device(dev.h, 0, C.c_void_p(dl.data_ptr()), C.c_void_p(dr.data_ptr()), W, H,
               C.byref(cfg), C.byref(fc), C.c_void_p(o.data_ptr()), C.c_void_p(dd.data_ptr()), 0), dev.h)
    stk._raise(L.stk_frame_wait(dev.h, 0, None, None, None), dev.h)
torch.cuda.synchronize()
print("ok")
