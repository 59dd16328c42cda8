"""Python mirror of the reference's stereotk stage/pipeline API, over the C-ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/stereotk/*.hpp so tests read like the
reference's own doctest suite; every compute call runs the sm_100a kernels of
libstk_b200.so (there is no CPU path -- without a B200 ``Device()`` raises).

Images are numpy arrays: RGB (h, w, 3) uint8, gray/mask (h, w) uint8, labels
(h, w) uint16, disparity (h, w) int16 with -1 = unknown.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (STK_ECUDA, STK_EFORMAT, STK_EIO, STK_EPARAM, STK_OK, StkConfig, StkFocus,
                   StkFrameInfo, StkFrameOut, StkStats, StkTimes)

UNKNOWN = -1  # DisparityMap::kUnknown (stereo.hpp:14)


class ParamError(ValueError):
    """stereotk::ParamError (error.hpp:19-21)."""


class IoError(RuntimeError):
    """stereotk::IoError (error.hpp:9-11)."""


class FormatError(RuntimeError):
    """stereotk::FormatError (error.hpp:14-16)."""


class CudaError(RuntimeError):
    """CUDA / device failure (no CPU fallback exists)."""


def _raise(rc: int, ctx=None) -> None:
    if rc == STK_OK:
        return
    msg = _lib.lib().stk_last_error(ctx)
    msg = msg.decode() if msg else ""
    if rc == STK_EPARAM:
        raise ParamError(msg)
    if rc == STK_EIO:
        raise IoError(msg)
    if rc == STK_EFORMAT:
        raise FormatError(msg)
    if rc == STK_ECUDA:
        raise CudaError(msg)
    raise RuntimeError(msg or f"stk error {rc}")


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ----------------------------------------------------------- value types --
@dataclass
class PipelineConfig:
    """stereotk::PipelineConfig (pipeline.hpp:18-25)."""
    k: int = 10
    window: int = 9
    max_disparity: int = 16
    threshold: int = 1
    prune_fraction: float = 0.04
    workers: int = 1

    def c(self) -> StkConfig:
        return StkConfig(self.k, self.window, self.max_disparity, self.threshold,
                         float(self.prune_fraction), self.workers)


@dataclass
class FocusSpec:
    """stereotk::FocusSpec (refocus.hpp:23-26) + the exact-blur switch."""
    ranges: Sequence = ()
    sigma: float = 2.0
    exact_blur: bool = False


@dataclass
class MatchConfig:
    """stereotk::MatchConfig (stereo.hpp:42-45)."""
    window: int = 9
    max_disparity: int = 16


@dataclass
class EvalResult:
    """stereotk::EvalResult (evaluate.hpp:10-16)."""
    bad_pixel_rate: float = 0.0
    compared: int = 0
    excluded: int = 0
    delta_d: float = 0.0


@dataclass
class Clustering:
    """stereotk::Clustering (segmentation.hpp:27-33)."""
    centers: np.ndarray
    bin_assignment: np.ndarray
    iterations_run: int

    def k(self) -> int:
        return len(self.centers)


@dataclass
class ComponentTable:
    """stereotk::ComponentTable (boundary.hpp:39-45)."""
    labels: np.ndarray
    sizes: np.ndarray
    by_size: np.ndarray


@dataclass
class GaussianKernel:
    """stereotk::GaussianKernel (refocus.hpp:11-20)."""
    size: int
    weights: np.ndarray  # (size, size) float64

    def at(self, i: int, j: int) -> float:
        h = self.size // 2
        return float(self.weights[i + h, j + h])


@dataclass
class StageTimes:
    """stereotk::StageTimes (pipeline.hpp:28-39) + blur; device milliseconds."""
    convert: float = 0.0
    segment: float = 0.0
    boundary: float = 0.0
    match: float = 0.0
    fill: float = 0.0
    peek: float = 0.0
    blur: float = 0.0

    def total(self) -> float:
        return self.convert + self.segment + self.boundary + self.match + self.fill + self.peek


@dataclass
class DepthStats:
    """stereotk::DepthStats (pipeline.hpp:42-49)."""
    pixels: int = 0
    boundary_raw: int = 0
    boundary_refined: int = 0
    matched: int = 0
    matched_fraction: float = 0.0
    known_fraction: float = 0.0


@dataclass
class DepthResult:
    """stereotk::DepthResult (pipeline.hpp:53-65)."""
    left_lightness: np.ndarray = None
    right_lightness: np.ndarray = None
    clustering: Clustering = None
    labels: np.ndarray = None
    boundary_raw: np.ndarray = None
    boundary_refined: np.ndarray = None
    boundary_anchored: np.ndarray = None
    sparse: np.ndarray = None
    row_filled: np.ndarray = None
    dense: np.ndarray = None
    stats: DepthStats = field(default_factory=DepthStats)
    info: dict = field(default_factory=dict)


# ---------------------------------------------------------------- device --
class Device:
    """One C-ABI context (one GPU, ``slots`` frames in flight)."""

    def __init__(self, device: int = 0, max_width: int = 0, max_height: int = 0, slots: int = 1):
        L = _lib.lib()
        h = C.c_void_p()
        _raise(L.stk_create(device, max_width, max_height, slots, C.byref(h)), None)
        self.h = h
        self.slots = slots
        self.device = device

    def close(self) -> None:
        if self.h:
            _lib.lib().stk_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_sad_kernel(self, kernel: str) -> None:
        _raise(_lib.lib().stk_set_sad_kernel(self.h, {"auto": 0, "list": 1, "strip": 2, "ws": 3}[kernel]),
               self.h)

    def set_use_graphs(self, on: bool) -> None:
        _raise(_lib.lib().stk_set_use_graphs(self.h, 1 if on else 0), self.h)

    def stream(self, slot: int = 0) -> int:
        return _lib.lib().stk_slot_stream(self.h, slot) or 0

    def _call(self, name, *args):
        _raise(getattr(_lib.lib(), name)(self.h, *args), self.h)


_tls = threading.local()


def default_device() -> Device:
    dev = getattr(_tls, "dev", None)
    if dev is None:
        dev = Device(0)
        _tls.dev = dev
    return dev


def _dev(device: Optional[Device]) -> Device:
    return device if device is not None else default_device()


def _c8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


# ----------------------------------------------------------- stage entries --
def rgb_to_lightness(image: np.ndarray, workers: int = 1, *, device=None) -> np.ndarray:
    """image.hpp:82 -- CIE L* rescaled to [0,255]."""
    image = _c8(image)
    h, w = image.shape[:2]
    out = np.empty((h, w), np.uint8)
    _dev(device)._call("stk_rgb_to_lightness", _p(image), w, h, _p(out))
    return out


def build_histogram(image: np.ndarray, workers: int = 1, *, device=None) -> np.ndarray:
    """segmentation.hpp:57 -> counts uint64[256]."""
    image = _c8(image)
    h, w = image.shape
    out = np.zeros(256, np.uint64)
    _dev(device)._call("stk_build_histogram", _p(image), w, h, _p(out))
    return out


def kmeans_histogram(histogram, k: int, max_iter: int = 100, tol: float = 0.5, *,
                     device=None) -> Clustering:
    """segmentation.hpp:67-68."""
    counts = np.ascontiguousarray(histogram, np.uint64)
    centers = np.zeros(max(k, 1), np.float64)
    asg = np.zeros(256, np.uint16)
    it = C.c_int(0)
    _dev(device)._call("stk_kmeans_histogram", _p(counts), k, max_iter, float(tol), _p(centers),
                       _p(asg), C.byref(it))
    return Clustering(centers[:k].copy(), asg, it.value)


def assign_pixels(image: np.ndarray, clustering: Clustering, *, device=None) -> np.ndarray:
    """segmentation.hpp:72."""
    image = _c8(image)
    h, w = image.shape
    asg = np.ascontiguousarray(clustering.bin_assignment, np.uint16)
    out = np.empty((h, w), np.uint16)
    _dev(device)._call("stk_assign_pixels", _p(image), w, h, _p(asg), clustering.k(), _p(out))
    return out


def detect_boundaries(labels: np.ndarray, workers: int = 1, *, device=None) -> np.ndarray:
    labels = np.ascontiguousarray(labels, np.uint16)
    h, w = labels.shape
    out = np.empty((h, w), np.uint8)
    _dev(device)._call("stk_detect_boundaries", _p(labels), w, h, _p(out))
    return out


def morph_fill(mask: np.ndarray, workers: int = 1, *, device=None) -> np.ndarray:
    mask = _c8(mask)
    h, w = mask.shape
    out = np.empty((h, w), np.uint8)
    _dev(device)._call("stk_morph_fill", _p(mask), w, h, _p(out))
    return out


def morph_remove(mask: np.ndarray, workers: int = 1, *, device=None) -> np.ndarray:
    mask = _c8(mask)
    h, w = mask.shape
    out = np.empty((h, w), np.uint8)
    _dev(device)._call("stk_morph_remove", _p(mask), w, h, _p(out))
    return out


def label_components(mask: np.ndarray, *, device=None) -> ComponentTable:
    mask = _c8(mask)
    h, w = mask.shape
    n = w * h
    labels = np.empty((h, w), np.int32)
    sizes = np.zeros(max(n, 1), np.uint32)
    bys = np.zeros(max(n, 1), np.int32)
    nc = C.c_int(0)
    _dev(device)._call("stk_label_components", _p(mask), w, h, _p(labels), _p(sizes), _p(bys),
                       max(n, 1), C.byref(nc))
    return ComponentTable(labels, sizes[: nc.value].copy(), bys[: nc.value].copy())


def prune_components(mask: np.ndarray, fraction: float, *, device=None) -> np.ndarray:
    mask = _c8(mask)
    h, w = mask.shape
    out = np.empty((h, w), np.uint8)
    _dev(device)._call("stk_prune_components", _p(mask), w, h, float(fraction), _p(out))
    return out


def add_border_anchors(mask: np.ndarray, margin: int, *, device=None) -> np.ndarray:
    mask = _c8(mask)
    h, w = mask.shape
    out = np.empty((h, w), np.uint8)
    _dev(device)._call("stk_add_border_anchors", _p(mask), w, h, margin, _p(out))
    return out


def sad_cost(left, right, x: int, y: int, d: int, window: int, *, device=None) -> int:
    left, right = _c8(left), _c8(right)
    h, w = left.shape
    out = C.c_uint32(0)
    _dev(device)._call("stk_sad_cost", _p(left), _p(right), w, h, x, y, d, window, C.byref(out))
    return out.value


def match_boundary_pixels(left, right, mask, config: MatchConfig = MatchConfig(),
                          workers: int = 1, *, device=None) -> np.ndarray:
    """stereo.hpp:58-62."""
    left, right, mask = _c8(left), _c8(right), _c8(mask)
    if left.shape != right.shape:
        raise ParamError("stereo: image sizes differ, left %dx%d vs right %dx%d"
                         % (left.shape[1], left.shape[0], right.shape[1], right.shape[0]))
    if mask.shape != left.shape:
        raise ParamError("stereo: mask size %dx%d does not match images %dx%d"
                         % (mask.shape[1], mask.shape[0], left.shape[1], left.shape[0]))
    h, w = left.shape
    out = np.empty((h, w), np.int16)
    _dev(device)._call("stk_match_boundary_pixels", _p(left), _p(right), _p(mask), w, h,
                       config.window, config.max_disparity, _p(out))
    return out


def dense_sad_baseline(left, right, config: MatchConfig = MatchConfig(), workers: int = 1, *,
                       device=None) -> np.ndarray:
    """evaluate.hpp:35-36: winner-takes-all SAD over every pixel with a valid window."""
    left, right = _c8(left), _c8(right)
    if left.shape != right.shape:
        raise ParamError("dense_sad_baseline: image sizes differ, left %dx%d vs right %dx%d"
                         % (left.shape[1], left.shape[0], right.shape[1], right.shape[0]))
    h, w = left.shape
    out = np.empty((h, w), np.int16)
    _dev(device)._call("stk_dense_sad_baseline", _p(left), _p(right), w, h, config.window,
                       config.max_disparity, _p(out))
    return out


def bad_pixel_rate(computed, truth, delta_d: float, workers: int = 1, *, device=None) -> EvalResult:
    """evaluate.hpp:22-24."""
    computed = np.ascontiguousarray(computed, np.int16)
    truth = np.ascontiguousarray(truth, np.int16)
    if computed.shape != truth.shape:
        raise ParamError("bad_pixel_rate: computed %dx%d vs truth %dx%d"
                         % (computed.shape[1], computed.shape[0], truth.shape[1], truth.shape[0]))
    h, w = computed.shape
    rate, cmp_, exc = C.c_double(0.0), C.c_uint64(0), C.c_uint64(0)
    _dev(device)._call("stk_bad_pixel_rate", _p(computed), _p(truth), w, h, float(delta_d),
                       C.byref(rate), C.byref(cmp_), C.byref(exc))
    return EvalResult(rate.value, cmp_.value, exc.value, float(delta_d))


def eval_report_json(result: EvalResult) -> str:
    """evaluate.cpp:220-227 (nlohmann::json::dump: keys sorted, compact)."""
    import json

    return json.dumps({"bad_pixel_rate": result.bad_pixel_rate, "compared": result.compared,
                       "delta_d": result.delta_d, "excluded": result.excluded},
                      separators=(",", ":"))


def probe_sad_peak(*, device=None) -> float:
    """Brute-force SAD ceiling of this device: VABSDIFF4 byte absolute
    differences per second from a register-only probe kernel."""
    out = C.c_double(0.0)
    _dev(device)._call("stk_probe_sad_peak", C.byref(out))
    return out.value


def fill_scanlines(sparse, workers: int = 1, *, device=None) -> np.ndarray:
    sparse = np.ascontiguousarray(sparse, np.int16)
    h, w = sparse.shape
    out = np.empty((h, w), np.int16)
    _dev(device)._call("stk_fill_scanlines", _p(sparse), w, h, _p(out))
    return out


def peek_columns(m, threshold: int, workers: int = 1, *, device=None) -> np.ndarray:
    m = np.ascontiguousarray(m, np.int16)
    h, w = m.shape
    out = np.empty((h, w), np.int16)
    _dev(device)._call("stk_peek_columns", _p(m), w, h, threshold, _p(out))
    return out


def default_kernel_size(sigma: float) -> int:
    return _lib.lib().stk_default_kernel_size(float(sigma))


def gaussian_kernel(sigma: float, size: int) -> GaussianKernel:
    wts = np.zeros(max(size, 1) ** 2, np.float64)
    _raise(_lib.lib().stk_gaussian_kernel(float(sigma), size, _p(wts)), None)
    return GaussianKernel(size, wts.reshape(size, size))


def _ranges(focus) -> tuple:
    rs = list(focus.ranges if isinstance(focus, FocusSpec) else focus)
    lo = np.array([r[0] for r in rs] or [0], np.int32)
    hi = np.array([r[1] for r in rs] or [0], np.int32)
    return lo, hi, len(rs)


def build_blur_map(depth, focus, max_disparity: int, *, device=None) -> np.ndarray:
    depth = np.ascontiguousarray(depth, np.int16)
    h, w = depth.shape
    lo, hi, n = _ranges(focus)
    out = np.empty((h, w), np.uint8)
    _dev(device)._call("stk_build_blur_map", _p(depth), w, h, _p(lo), _p(hi), n, max_disparity,
                       _p(out))
    return out


def selective_blur(image, blur_map, kernel: GaussianKernel, workers: int = 1, *, sigma=None,
                   exact: bool = False, device=None) -> np.ndarray:
    """refocus.hpp:50-51.  The kernel is regenerated on the device side from
    (sigma, size); pass ``sigma`` when ``kernel`` came from elsewhere."""
    image, blur_map = _c8(image), _c8(blur_map)
    h, w = image.shape[:2]
    if blur_map.shape != (h, w):
        raise ParamError("selective_blur: blur map %dx%d does not match image %dx%d"
                         % (blur_map.shape[1], blur_map.shape[0], w, h))
    s = sigma if sigma is not None else getattr(kernel, "sigma", None)
    if s is None:
        raise ParamError("selective_blur: sigma unknown for this kernel")
    out = np.empty_like(image)
    _dev(device)._call("stk_selective_blur", _p(image), _p(blur_map), w, h, float(s),
                       kernel.size, 1 if exact else 0, _p(out))
    return out


def validate_config(config: PipelineConfig) -> None:
    c = config.c()
    _raise(_lib.lib().stk_validate_config(C.byref(c)), None)


# --------------------------------------------------------------- pipeline --
def _focus_c(focus: Optional[FocusSpec], kernel_size: int):
    if focus is None:
        return None, None
    lo, hi, n = _ranges(focus)
    f = StkFocus(lo.ctypes.data_as(C.POINTER(C.c_int)), hi.ctypes.data_as(C.POINTER(C.c_int)), n,
                 float(focus.sigma), int(kernel_size), 1 if focus.exact_blur else 0)
    return f, (lo, hi)


def _check_pair(left, right):
    if left.shape != right.shape:
        raise ParamError("pipeline: image sizes differ, left %dx%d vs right %dx%d"
                         % (left.shape[1], left.shape[0], right.shape[1], right.shape[0]))


def _run(left, right, config, focus, kernel_size, full, times, device):
    left, right = _c8(left), _c8(right)
    _check_pair(left, right)
    h, w = left.shape[:2]
    dev = _dev(device)
    r = DepthResult()
    r.dense = np.empty((h, w), np.int16)
    out = StkFrameOut()
    out.dense = _p(r.dense)
    refocused = None
    if focus is not None:
        refocused = np.empty((h, w, 3), np.uint8)
        out.refocused = _p(refocused)
    centers = np.zeros(256, np.float64)
    asg = np.zeros(256, np.uint16)
    if full:
        r.left_lightness = np.empty((h, w), np.uint8)
        r.right_lightness = np.empty((h, w), np.uint8)
        r.labels = np.empty((h, w), np.uint16)
        r.boundary_raw = np.empty((h, w), np.uint8)
        r.boundary_refined = np.empty((h, w), np.uint8)
        r.boundary_anchored = np.empty((h, w), np.uint8)
        r.sparse = np.empty((h, w), np.int16)
        r.row_filled = np.empty((h, w), np.int16)
        for name in ("left_lightness", "right_lightness", "labels", "boundary_raw",
                     "boundary_refined", "boundary_anchored", "sparse", "row_filled"):
            setattr(out, name, _p(getattr(r, name)))
        out.centers = _p(centers)
        out.bin_assignment = _p(asg)
    cfg = config.c()
    fc, keep = _focus_c(focus, kernel_size)
    st = StkStats()
    tm = StkTimes()
    info = StkFrameInfo()
    L = _lib.lib()
    _raise(L.stk_frame_submit(dev.h, 0, _p(left), _p(right), w, h, C.byref(cfg),
                              C.byref(fc) if fc is not None else None, C.byref(out),
                              1 if times is not None else 0), dev.h)
    _raise(L.stk_frame_wait(dev.h, 0, C.byref(st), C.byref(tm), C.byref(info)), dev.h)
    r.stats = DepthStats(st.pixels, st.boundary_raw, st.boundary_refined, st.matched,
                         st.matched_fraction, st.known_fraction)
    r.info = dict(sad_ops=info.sad_ops, components=info.components, k=info.k,
                  iterations_run=info.iterations_run, kernels=info.kernels, graph=info.graph)
    if full:
        r.clustering = Clustering(centers[: info.k].copy(), asg, info.iterations_run)
    if times is not None:
        for n in ("convert", "segment", "boundary", "match", "fill", "peek", "blur"):
            setattr(times, n, getattr(tm, n))
    return r, refocused


def run_depth_pipeline(left, right, config: PipelineConfig = PipelineConfig(),
                       times: Optional[StageTimes] = None, *, full: bool = True,
                       device=None) -> DepthResult:
    """pipeline.hpp:78-80.  ``full=False`` skips the intermediates (lean mode)."""
    return _run(left, right, config, None, 0, full, times, device)[0]


def run_refocus_pipeline(left, right, config: PipelineConfig, focus: FocusSpec,
                         kernel_size: int = 0, depth_out: Optional[list] = None, *,
                         device=None) -> np.ndarray:
    """pipeline.hpp:85-89.  ``depth_out``, when a list, receives the DepthResult."""
    r, out = _run(left, right, config, focus, kernel_size, depth_out is not None, None, device)
    if depth_out is not None:
        depth_out.append(r)
    return out


# ------------------------------------------------------------- file I/O --
# image.hpp:55-79, evaluate.hpp:27-67, tools/main.cpp:247-284 -- host code in
# libstk_b200.so (csrc/stk_io.cpp); no GPU needed.
def _b(path) -> bytes:
    return str(path).encode()


def _probe(path):
    w, h, c = C.c_int(), C.c_int(), C.c_int()
    _raise(_lib.lib().stk_image_probe(_b(path), C.byref(w), C.byref(h), C.byref(c)))
    return w.value, h.value, c.value


def load_image(path) -> np.ndarray:
    """image.hpp:55-60: PNG / P6 / P5 (replicated) as (h, w, 3) uint8."""
    w, h, _ = _probe(path)
    out = np.empty((h, w, 3), np.uint8)
    _raise(_lib.lib().stk_load_image(_b(path), _p(out), w, h))
    return out


def load_gray(path, comments: Optional[list] = None) -> np.ndarray:
    """image.hpp:62-67: P5 or grey PNG as (h, w) uint8; header comments appended to ``comments``."""
    w, h, _ = _probe(path)
    out = np.empty((h, w), np.uint8)
    need = C.c_size_t()
    buf = C.create_string_buffer(4096)
    L = _lib.lib()
    _raise(L.stk_load_gray(_b(path), _p(out), w, h, buf, 4096, C.byref(need)))
    if need.value > 4096:
        buf = C.create_string_buffer(need.value)
        _raise(L.stk_load_gray(_b(path), _p(out), w, h, buf, need.value, C.byref(need)))
    if comments is not None:
        comments.extend(buf.value.decode(errors="replace").splitlines())
    return out


def save_gray(image: np.ndarray, path, comments: Sequence[str] = ()) -> None:
    """image.hpp:69-72 (binary PGM, comments after the magic number)."""
    img = _c8(image)
    text = "".join(c + "\n" for c in comments).encode() if comments else None
    _raise(_lib.lib().stk_save_gray(_b(path), _p(img), img.shape[1], img.shape[0], text))


def save_rgb(image: np.ndarray, path) -> None:
    """image.hpp:74-76 (.png -> PNG, anything else -> binary PPM)."""
    img = _c8(image)
    _raise(_lib.lib().stk_save_rgb(_b(path), _p(img), img.shape[1], img.shape[0]))


def save_disparity(m: np.ndarray, path, output_scale: float) -> None:
    """evaluate.hpp:53-58: PGM of round(d * scale) + '# scale' comment + sibling mask."""
    d = np.ascontiguousarray(m, dtype=np.int16)
    _raise(_lib.lib().stk_save_disparity(_b(path), _p(d), d.shape[1], d.shape[0], float(output_scale)))


def load_disparity(path, fallback_scale: float = 0.0) -> np.ndarray:
    """evaluate.hpp:63-67."""
    w, h, _ = _probe(path)
    out = np.empty((h, w), np.int16)
    _raise(_lib.lib().stk_load_disparity(_b(path), _p(out), w, h, float(fallback_scale)))
    return out


def load_ground_truth(path, scale: float) -> np.ndarray:
    """evaluate.hpp:27-30: value / scale rounded, 0 -> unknown."""
    if not scale > 0.0:  # checked before the file is touched, as evaluate.cpp:76-80
        _raise(_lib.lib().stk_load_ground_truth(_b(path), None, 0, 0, float(scale)))
    w, h, _ = _probe(path)
    out = np.empty((h, w), np.int16)
    _raise(_lib.lib().stk_load_ground_truth(_b(path), _p(out), w, h, float(scale)))
    return out


def disparity_mask_path(path) -> str:
    """evaluate.hpp:60-61."""
    need = C.c_size_t()
    buf = C.create_string_buffer(len(str(path).encode()) + 64)
    _raise(_lib.lib().stk_disparity_mask_path(_b(path), buf, len(buf), C.byref(need)))
    return buf.value.decode()


def list_frame_pairs(directory) -> list:
    """tools/main.cpp:247-284: [(left, right)] for every <stem>_L/_R pair, by stem."""
    need, n = C.c_size_t(), C.c_int()
    L = _lib.lib()
    _raise(L.stk_list_frame_pairs(_b(directory), None, 0, C.byref(need), C.byref(n)))
    buf = C.create_string_buffer(need.value)
    _raise(L.stk_list_frame_pairs(_b(directory), buf, need.value, C.byref(need), C.byref(n)))
    return [tuple(line.split("\t")) for line in buf.value.decode().splitlines()]


def load_frames(directory) -> list:
    """The CLI's load_frames: [(left_rgb, right_rgb)] in stem order."""
    return [(load_image(l), load_image(r)) for l, r in list_frame_pairs(directory)]


@dataclass
class VideoReport:
    """stk_video_report: what one refocus_video call did and how fast."""
    frames: int
    frames_total: int
    wall_s: float
    frames_per_s: float
    decode_s: float
    write_s: float
    gpu_wait_s: float
    matched_fraction: float


def refocus_video(in_dir, out_dir, config: PipelineConfig, focus: FocusSpec, kernel_size: int = 0, *,
                  slots: int = 0, decode_threads: int = 4, write_threads: int = 2, png: bool = False,
                  disparity_scale: float = 0.0, shard_index: int = 0, shard_count: int = 1,
                  device: Optional[Device] = None) -> VideoReport:
    """Every <stem>_L/_R pair of ``in_dir`` refocused into ``out_dir`` with
    decode, copies, kernels and encode overlapped (stk_video_refocus).
    ``slots`` = GPU frames in flight (default: all of the device's)."""
    from ._lib import StkVideoOpts, StkVideoReport

    dev = _dev(device)
    slots = slots or dev.slots
    cfg = config.c()
    fc, keep = _focus_c(focus, kernel_size)
    opts = StkVideoOpts(slots, decode_threads, write_threads, 1 if png else 0, float(disparity_scale),
                        shard_index, shard_count)
    rep = StkVideoReport()
    _raise(_lib.lib().stk_video_refocus(dev.h, _b(in_dir), _b(out_dir), C.byref(cfg), C.byref(fc),
                                        C.byref(opts), C.byref(rep)), None)
    return VideoReport(rep.frames, rep.frames_total, rep.wall_s, rep.frames_per_s, rep.decode_s,
                       rep.write_s, rep.gpu_wait_s, rep.matched_fraction)
