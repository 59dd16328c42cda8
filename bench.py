"""bench.py -- 4096x2304 stereo frames/s through the B200 depth + refocus path.

A "step" is one stereo frame pair taken through run_refocus_pipeline's work
(L*, histogram K-Means, boundary detect/fill/remove, CC prune + anchors, SAD
on the boundary list, row fill, column peek, depth-masked blur) on a G2 "dead
leaves" synthetic frame (~18-19 % boundary pixels).

  value : frames/s with the input pair already resident in HBM (a pool of P
          distinct frames, 8 x 56.6 MB > L2, cycled), S frames in flight.
  e2e   : the same through the C-ABI's host-pointer entry (stk_frame_submit):
          pinned host RGB pair H2D, refocused RGB + dense disparity D2H inside
          the timed region, S frames in flight.
  --impl reference : the reference's own CPU implementation (oracle/_ref,
          compiled from /root/reference sources; else the C port) on the host
          cores, rank 0 only.

Multi-GPU (torchrun): frames are sharded by index, frame f -> rank f % N
(shard.shard_frames), no collective on the data path ("scaling": "weak");
gloo (CPU) carries only the barrier and the max-over-ranks of the device
time -- NCCL is never initialised.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (W, H, D, window, K, focus ranges, sigma)
    "A": (450, 375, 16, 9, 4, [(8, 16)], 2.0),
    "B": (1920, 1080, 64, 15, 6, [(32, 64)], 2.0),
    "C": (4096, 2304, 128, 21, 8, [(64, 128)], 2.0),
    "E": (7680, 4320, 256, 31, 8, [(128, 256)], 8.0),
}
METRIC = "4096x2304 stereo frames/sec end-to-end (per-stage HBM GB/s in roofline_stages)"


def workload(cfgname):
    """The workload string both arms print (identical config => same_config)."""
    W, H, D, win, K, focus, sigma = CONFIGS[cfgname]
    return (f"{W}x{H} G2 dead-leaves stereo video, D={D}, w={win}, K={K}, "
            f"focus={focus}, sigma={sigma}, threshold=1, prune=0.04")


class Control:
    """Control plane of the multi-GPU job: barrier and max-over-ranks over
    gloo (CPU).  No frame data crosses ranks and NCCL is never initialised:
    the path has no collective."""

    def __init__(self, world, rank):
        self.world, self.rank = world, rank
        self.dist = None
        if world > 1:
            import torch.distributed as dist

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("gloo", rank=rank, world_size=world)
            self.dist = dist

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def max(self, value):
        from paper_2001_07809_b200 import shard

        return shard.max_over_ranks(value, self.dist)

    def close(self):
        if self.dist is not None:
            self.dist.destroy_process_group()


class Job:
    """This rank's share of a weak-scaled run: `steps` frames per rank, global
    frame f -> rank f % world (shard.shard_frames); the frame pool holds this
    rank's first P frame indices (synthetic seed 2001 + f)."""

    def __init__(self, world, rank, steps, pool):
        from paper_2001_07809_b200 import shard

        self.world, self.rank, self.steps = world, rank, steps
        self.frames = shard.shard_frames(steps * world, rank, world)
        self.pool_ids = shard.shard_frames(max(1, pool) * world, rank, world)

    def pool_slot(self, i):
        """Pool entry used by this rank's i-th frame."""
        return i % len(self.pool_ids)


def timed_region(ctrl, sync, start, stop, submit, steps, drain):
    """W untimed warm-up frames happen before this.  Barrier + device sync on
    both sides; the device time of `steps` submits (start/stop return the
    event bracket, stop returns ms); the max over ranks is the job's time."""
    drain()
    sync()
    ctrl.barrier()
    start()
    for i in range(steps):
        submit(i)
    ms = stop()
    drain()
    sync()
    ms = ctrl.max(ms)
    ctrl.barrier()
    return ms


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=250)  # the paper's 250-frame video
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="C", choices=sorted(CONFIGS))
    p.add_argument("--pool", type=int, default=8, help="distinct synthetic frames cycled")
    p.add_argument("--slots", type=int, default=16, help="frames in flight per GPU")
    p.add_argument("--sad", default="auto", choices=["auto", "list", "strip"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample-s", type=float, default=20.0)
    p.add_argument("--cpu-serial", type=int, default=1, help="also time one reference frame at workers = 1")
    p.add_argument("--e2e-rgb-only", action="store_true",
                   help="e2e leg reads back only the refocused RGB (default: refocused RGB + dense "
                        "disparity, SURVEY.md 8(d))")
    return p.parse_args()


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                          f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout
                    f = [x.strip() for x in out.strip().split(",")]
                    if len(f) >= 7:
                        self.samples.append(f)
                except Exception:
                    pass
                self._stop.wait(0.05)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)
        if not self.samples:
            return None
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ------------------------------------------------------------- reference --
def reference_frames(cfgname, n, pool):
    from paper_2001_07809_b200 import synth

    W, H, D, win, K, focus, sigma = CONFIGS[cfgname]
    return [synth.dead_leaves(W, H, D, frame=i % pool) for i in range(min(n, pool))]


def run_reference_frame(ref, frame, cfgname, workers):
    W, H, D, win, K, focus, sigma = CONFIGS[cfgname]
    l, r = frame
    t0 = time.perf_counter()
    res = ref.run_frame(l, r, k=K, window=win, max_disparity=D, threshold=1,
                        prune_fraction=0.04, focus=focus, sigma=sigma, workers=workers)
    return time.perf_counter() - t0, res


def cpu_reference(cfgname, sample_s, warmup=1, steps=None, pool=8):
    """Time the reference CPU path on this host; returns (fps, cores, kind, sample)."""
    os.environ.setdefault("OMP_WAIT_POLICY", "passive")
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")
    import oracle

    ref = oracle.reference()
    kind = "reference"
    cores = os.cpu_count() or 1
    if ref is None:
        ref = oracle.port()
        kind = "port"
        cores = 1
    frames = reference_frames(cfgname, max(1, min(pool, 4)), pool)
    for i in range(warmup):
        run_reference_frame(ref, frames[i % len(frames)], cfgname, cores)
    times = []
    t_all = time.perf_counter()
    i = 0
    while True:
        dt, _ = run_reference_frame(ref, frames[i % len(frames)], cfgname, cores)
        times.append(dt)
        i += 1
        if steps is not None and i >= steps:
            break
        if steps is None and time.perf_counter() - t_all >= sample_s:
            break
        if steps is not None and time.perf_counter() - t_all >= 240.0:
            break  # bounded: report the rate over the frames done
    fps = len(times) / sum(times)
    W, H = CONFIGS[cfgname][:2]
    sample = (f"{len(times)} full {W}x{H} G2 frames (run_depth_pipeline + blur map + "
              f"gaussian_kernel + selective_blur), OMP {cores} threads "
              f"OMP_WAIT_POLICY={os.environ.get('OMP_WAIT_POLICY')}")
    return fps, cores, kind, sample, times


def impl_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    fps, cores, kind, sample, times = cpu_reference(args.config, None, warmup=args.warmup,
                                                    steps=args.steps, pool=args.pool)
    W, H, D, win, K, focus, sigma = CONFIGS[args.config]
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s",
        "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": 1e3 / fps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8/i16/f64", "data": "synthetic",
        "config": {"workload": workload(args.config), "frames_pool": args.pool},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------- B200 --
def main():
    args = parse()
    if args.impl == "reference":
        return impl_reference(args)

    import numpy as np
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # STK_BENCH_ONE_DEVICE=1: every rank on device 0 -- a functional check of
    # the multi-process path on a one-GPU box (ranks never wait on each
    # other's kernels, only on the gloo barrier); its throughput is not a
    # scaling number
    if os.environ.get("STK_BENCH_ONE_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    all_cpus = os.sched_getaffinity(0)
    affinity = _pin_near_gpu(torch, local)  # host thread near the GPU's PCIe root
    ctrl = Control(world, rank)  # gloo: barrier + max over ranks; no NCCL, no data collective

    from paper_2001_07809_b200 import _lib, synth
    from paper_2001_07809_b200 import stereotk as stk

    W, H, D, win, K, focus, sigma = CONFIGS[args.config]
    N = W * H
    S = max(1, args.slots)
    dev = stk.Device(local, W, H, slots=S)
    dev.set_sad_kernel(args.sad)
    L = _lib.lib()
    cfg = stk.PipelineConfig(k=K, window=win, max_disparity=D, threshold=1, prune_fraction=0.04)
    c_cfg = cfg.c()
    fspec = stk.FocusSpec(ranges=focus, sigma=sigma)
    c_focus, _keep = stk._focus_c(fspec, 0)

    # frame pool: this rank's first P global frame indices (f = rank + i * world)
    job = Job(world, rank, args.steps, args.pool)
    P = len(job.pool_ids)
    frames = [synth.dead_leaves(W, H, D, frame=f) for f in job.pool_ids]
    d_in = [(torch.from_numpy(l).cuda(), torch.from_numpy(r).cuda()) for l, r in frames]
    d_out = [(torch.empty((H, W, 3), dtype=torch.uint8, device="cuda"),
              torch.empty((H, W), dtype=torch.int16, device="cuda")) for _ in range(S)]
    streams = [torch.cuda.ExternalStream(dev.stream(s)) for s in range(S)]

    def check(rc):
        stk._raise(rc, dev.h)

    info = _lib.StkFrameInfo()
    inflight = [False] * S

    def wait(slot, want_info=False):
        if inflight[slot]:
            check(L.stk_frame_wait(dev.h, slot, None, None, C.byref(info) if want_info else None))
            inflight[slot] = False

    def drain():
        for s in range(S):
            wait(s)

    def submit_device(i):
        slot = i % S
        wait(slot)
        l, r = d_in[job.pool_slot(i)]
        o, dd = d_out[slot]
        check(L.stk_frame_submit_device(dev.h, slot, C.c_void_p(l.data_ptr()),
                                        C.c_void_p(r.data_ptr()), W, H, C.byref(c_cfg),
                                        C.byref(c_focus), C.c_void_p(o.data_ptr()),
                                        C.c_void_p(dd.data_ptr()), 0))
        inflight[slot] = True

    # CUDA events: start on slot 0's stream (every slot stream waits on it),
    # end on slot 0's stream after joining every slot stream
    ev = {}

    def start():
        ev["0"] = torch.cuda.Event(enable_timing=True)
        ev["1"] = torch.cuda.Event(enable_timing=True)
        ev["0"].record(streams[0])
        for s in range(1, S):
            streams[s].wait_event(ev["0"])

    def stop():
        for s in range(1, S):
            e = torch.cuda.Event()
            e.record(streams[s])
            streams[0].wait_event(e)
        ev["1"].record(streams[0])
        ev["1"].synchronize()
        return ev["0"].elapsed_time(ev["1"])

    sync = torch.cuda.synchronize

    # ---- warm-up (also builds the per-slot CUDA graphs: at least one untimed
    # frame per slot so no graph is captured inside the timed region)
    n_warm = max(3, args.warmup, S)
    for i in range(n_warm):
        submit_device(i)
    for s in range(S):
        wait(s, want_info=True)
    kernels_per_frame = info.kernels

    # ---- device-resident timed region
    clocks = ClockSampler(local)
    clocks.start()
    ms_dev = timed_region(ctrl, sync, start, stop, submit_device, args.steps, drain)
    clk = clocks.stop()
    fps_dev = world * args.steps / (ms_dev / 1e3)

    # ---- end-to-end through the host-pointer C-ABI entry (pinned buffers):
    # H2D of the RGB pair, D2H of the refocused RGB + dense disparity
    dense_back = not args.e2e_rgb_only
    hp = []
    for i in range(P):
        l, r = frames[i]
        bl = np.frombuffer((C.c_uint8 * (3 * N)).from_address(_pinned(L, 3 * N)), np.uint8)
        br = np.frombuffer((C.c_uint8 * (3 * N)).from_address(_pinned(L, 3 * N)), np.uint8)
        bl[:] = l.reshape(-1)
        br[:] = r.reshape(-1)
        hp.append((bl, br))
    ho = []
    for s in range(S):
        o = np.frombuffer((C.c_uint8 * (3 * N)).from_address(_pinned(L, 3 * N)), np.uint8)
        dd = np.frombuffer((C.c_int16 * N).from_address(_pinned(L, 2 * N)), np.int16)
        ho.append((o, dd))
    outs = [_lib.StkFrameOut() for _ in range(S)]
    for s in range(S):
        outs[s].refocused = ho[s][0].ctypes.data
        outs[s].dense = ho[s][1].ctypes.data if dense_back else None

    def submit_host(i):
        slot = i % S
        wait(slot)
        bl, br = hp[job.pool_slot(i)]
        check(L.stk_frame_submit(dev.h, slot, C.c_void_p(bl.ctypes.data),
                                 C.c_void_p(br.ctypes.data), W, H, C.byref(c_cfg),
                                 C.byref(c_focus), C.byref(outs[slot]), 0))
        inflight[slot] = True

    for i in range(n_warm):
        submit_host(i)
    ms_e2e = timed_region(ctrl, sync, start, stop, submit_host, args.steps, drain)
    fps_e2e = world * args.steps / (ms_e2e / 1e3)
    h2d_bytes = 2 * 3 * N
    d2h_bytes = 3 * N + (2 * N if dense_back else 0)
    for s in range(S):
        wait(s)
    pcie = _pcie_probe(local)

    # ---- per-stage device times (separate, event-instrumented frames)
    stage_ms = {}
    infos = []
    n_stage = 5
    tm = _lib.StkTimes()
    for i in range(n_stage):
        l, r = d_in[i % P]
        o, dd = d_out[0]
        wait(0)
        check(L.stk_frame_submit_device(dev.h, 0, C.c_void_p(l.data_ptr()),
                                        C.c_void_p(r.data_ptr()), W, H, C.byref(c_cfg),
                                        C.byref(c_focus), C.c_void_p(o.data_ptr()),
                                        C.c_void_p(dd.data_ptr()), 1))
        st = _lib.StkStats()
        check(L.stk_frame_wait(dev.h, 0, C.byref(st), C.byref(tm), C.byref(info)))
        for k in ("convert", "segment", "boundary", "match", "fill", "peek", "blur"):
            stage_ms.setdefault(k, []).append(getattr(tm, k))
        infos.append((st.matched, info.sad_ops, st.matched_fraction))
    stage_ms = {k: statistics.median(v) for k, v in stage_ms.items()}
    M = statistics.mean(x[0] for x in infos)
    sad_ops = statistics.mean(x[1] for x in infos)
    matched_frac = statistics.mean(x[2] for x in infos)

    # algorithmic HBM bytes per stage, per frame
    alg = {"convert": 8 * N, "segment": N, "boundary": 12 * N + 4 * M, "match": 4 * N + 4 * M,
           "fill": 4 * N, "peek": 4 * N, "blur": 8 * N}
    peaks = _peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    stages = {}
    for k, b in alg.items():
        t = stage_ms[k]
        gbs = b / (t * 1e-3) / 1e9 if t > 0 else None
        stages[k] = {"ms": round(t, 4), "alg_bytes": int(b),
                     "GB/s": round(gbs, 1) if gbs else None,
                     "frac_hbm": round(gbs / hbm_peak, 4) if gbs else None}
    stages["match"]["byte_sad_per_s"] = sad_ops / (stage_ms["match"] * 1e-3)
    total_alg = sum(alg.values())
    frame_ms_dev = ms_dev / args.steps
    dominant = max(stage_ms, key=stage_ms.get)
    peak_src = ("MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks else
                "fallback 6650 GB/s (B200_PROFILING.md)")
    # dominant kernel: the match stage is one launch (K5c k_sad_ws); algorithmic
    # bytes per launch = 4N + 4M; CUDA-event time on its stream
    prof = _ncu_profile()
    sad_prof = next((v[-1] for k, v in prof.items() if "sad_ws" in k or "sad_strip" in k), {})
    traffic = (sad_prof.get("dram_read_bytes", 0) + sad_prof.get("dram_write_bytes", 0)) or None
    t_match = stage_ms["match"] * 1e-3
    roofline = {
        "bound": "hbm", "kernel": "k_sad_ws (match stage, one launch per frame)",
        "achieved": round(alg["match"] / t_match / 1e9, 1), "peak": hbm_peak, "unit": "GB/s",
        "frac": round(alg["match"] / t_match / 1e9 / hbm_peak, 4),
        "traffic": traffic, "alg_bytes": int(alg["match"]),
        "peak_source": peak_src,
        "note": "SAD is integer-ALU bound (VABSDIFF4/PRMT/IADD3; no tensor cores per the north "
                "star): its HBM fraction is small by construction; alu_pipe_pct is the binding "
                "resource (ncu, profiles/)",
        "byte_sad_per_s": sad_ops / t_match,
        "alu_pipe_pct_active": sad_prof.get("alu_pipe_pct_active"),
        "shared_wavefronts_pct": sad_prof.get("lsu_shared_wavefronts_pct"),
        "traffic_source": "profiles/r02_ncu_kernels.json (ncu --set full, one 4K launch)" if traffic else None,
    }
    # the brute-force SAD ceiling (VABSDIFF4 issue rate,
    # microbenchmarked here) and the frame roofline 1 / (bytes/BW + SAD/peak)
    sad_peak = C.c_double(0.0)
    if L.stk_probe_sad_peak(dev.h, C.byref(sad_peak)) == 0 and sad_peak.value > 0:
        roofline["sad_ceiling_byte_ad_per_s"] = sad_peak.value
        roofline["byte_sad_vs_ceiling"] = round(sad_ops / t_match / sad_peak.value, 3)
        roofline["ceiling_note"] = ("ceiling = measured VABSDIFF4 rate x 4 (brute-force w^2 per "
                                    "(pixel, d)); the box-filter formulation exceeds it")
    roofline_frame = {
        "bound": "hbm", "kernel": "frame (all launches, algorithmic 41N+8M bytes)",
        "achieved": round(total_alg / (frame_ms_dev * 1e-3) / 1e9, 1), "peak": hbm_peak, "unit": "GB/s",
        "frac": round(total_alg / (frame_ms_dev * 1e-3) / 1e9 / hbm_peak, 4), "dominant_stage": dominant,
    }
    if sad_peak.value > 0:
        model_fps = 1.0 / (total_alg / 8.0e12 + sad_ops / sad_peak.value)
        roofline_frame["survey_model_fps"] = round(model_fps, 1)
        roofline_frame["fps_vs_survey_model"] = round(fps_dev / model_fps, 3)

    line = {
        "metric": METRIC, "value": round(fps_dev, 3), "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_dev / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u8/i16 (int stages), f64 (L*, K-Means), f32-accumulated blur (f16 hi/lo tensor-core products)", "data": "synthetic",
        "config": {"workload": workload(args.config),
                   "frames_pool": P, "frames_in_flight": S, "warmup_frames": n_warm,
                   "l2": "inputs larger than L2 (pool of distinct frames, ~56.6 MB each)",
                   "parallelism": f"frame-sharded x{world} (frame f -> rank f % {world}, no NCCL)",
                   "sad_kernel": args.sad, "matched_fraction": round(matched_frac, 4)},
        "e2e": {"value": round(fps_e2e, 3), "unit": "frames/s",
                "h2d_bytes_per_step": h2d_bytes,
                "d2h_bytes_per_step": d2h_bytes,
                "path": "stk_frame_submit (C-ABI, pinned host buffers)",
                "pcie": _pcie_model(pcie, h2d_bytes, d2h_bytes,
                                    fps_e2e / world, frame_ms_dev)},
        "gpu_launches": int(kernels_per_frame * args.steps * 2),
        "kernels_per_frame": int(kernels_per_frame),
        "gpu_launches_note": "kernels_per_frame x steps in each of the two timed regions (device-resident, e2e)",
        "roofline": roofline,
        "roofline_frame": roofline_frame,
        "roofline_stages": stages,
        "sad_ops_per_frame": int(sad_ops),
        "host_affinity": affinity,
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        os.sched_setaffinity(0, all_cpus)  # the CPU baseline gets every host core
        fps, cores, kind, sample, _ = cpu_reference(args.config, args.cpu_sample_s, warmup=0,
                                                    pool=args.pool)
        line["cpu_baseline"] = {"value": fps, "unit": "frames/s", "cores": cores, "kind": kind,
                                "sample": sample, "cpu_model": _cpu_model(), "nproc": os.cpu_count()}
        if kind == "reference" and args.cpu_serial:
            # the reference at workers = 1 as well (one frame, bounded)
            ref = __import__("oracle").reference()
            frame = reference_frames(args.config, 1, 1)[0]
            dt, _ = run_reference_frame(ref, frame, args.config, 1)
            line["cpu_baseline"]["serial"] = {"value": 1.0 / dt, "unit": "frames/s", "cores": 1,
                                              "sample": "1 frame, workers = 1"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    dev.close()
    ctrl.close()
    return 0


def _pin_near_gpu(torch, local):
    """Best effort: bind this rank to the CPUs of the NUMA node the GPU hangs
    off (its PCIe root), before any pinned host buffer is touched, so staging
    memory is node-local.  Returns a description for the JSON line."""
    try:
        p = torch.cuda.get_device_properties(local)
        bus = "%04x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
        base = "/sys/bus/pci/devices/" + bus
        node = int(open(base + "/numa_node").read().strip())
        cpus_txt = open(base + "/local_cpulist").read().strip()
        cpus = set()
        for part in cpus_txt.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        cpus &= os.sched_getaffinity(0)
        if cpus and len(cpus) < os.cpu_count():
            os.sched_setaffinity(0, cpus)
            return {"gpu_pci": bus, "numa_node": node, "cpus": cpus_txt}
        return {"gpu_pci": bus, "numa_node": node, "cpus": "all (single node)"}
    except (OSError, ValueError, AttributeError):
        return None


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


_pinned_keep = []


def _pinned(L, nbytes):
    p = C.c_void_p()
    rc = L.stk_host_alloc(nbytes, C.byref(p))
    if rc != 0:
        raise RuntimeError("pinned alloc failed")
    _pinned_keep.append(p)
    return p.value


def _pcie_probe(dev_index, mb=128, reps=5):
    """Pinned host <-> device copy bandwidth on this box (GB/s): H2D alone,
    D2H alone, and both directions at once on two streams (the e2e leg's
    ceiling: a frame's inputs go up while an earlier frame's result comes down)."""
    import torch

    n = mb << 20
    h_a = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_b = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(n, dtype=torch.uint8, device=f"cuda:{dev_index}")
    d_b = torch.empty(n, dtype=torch.uint8, device=f"cuda:{dev_index}")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        # the copies run on s1/s2: join them into the current stream before e1
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e-3

    def h2d():
        with torch.cuda.stream(s1):
            d_a.copy_(h_a, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)

    def d2h():
        with torch.cuda.stream(s2):
            h_b.copy_(d_b, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s2)

    def both():
        with torch.cuda.stream(s1):
            d_a.copy_(h_a, non_blocking=True)
        with torch.cuda.stream(s2):
            h_b.copy_(d_b, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)

    t_h = timed(h2d)
    t_d = timed(d2h)
    t_b = timed(both)
    gb = reps * n / 1e9
    return {"h2d_GBps": round(gb / t_h, 1), "d2h_GBps": round(gb / t_d, 1),
            "duplex_GBps_each_way": round(gb / t_b, 1), "probe": f"{reps} x {mb} MiB pinned copies"}


def _pcie_model(pcie, h2d_bytes, d2h_bytes, fps_e2e, frame_ms_dev):
    """e2e ceiling: per frame max(H2D time, D2H time, device time) with the
    copies overlapping each other (duplex bandwidth) and the kernels."""
    bw = pcie["duplex_GBps_each_way"] * 1e9
    t = max(h2d_bytes / bw, d2h_bytes / bw, frame_ms_dev * 1e-3)
    out = dict(pcie)
    out["achieved_h2d_GBps"] = round(h2d_bytes * fps_e2e / 1e9, 1)
    out["model_fps"] = round(1.0 / t, 1)
    out["frac"] = round(fps_e2e * t, 3)
    return out


def _ncu_profile():
    """Per-kernel ncu summary committed under profiles/ (scripts/ncu_to_json.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_ncu_kernels.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


if __name__ == "__main__":
    sys.exit(main())
