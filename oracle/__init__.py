"""oracle -- TEST INFRASTRUCTURE ONLY.

ctypes bindings to
  * ``liboracle.so``        -- the C restatement of the reference path
                               (oracle/stk_oracle.c, "port"), and
  * ``_ref/libstk_ref.so``  -- the unmodified reference sources compiled by
                               oracle/Makefile plus an extern "C" adapter
                               (oracle/ref_capi.cpp, "reference").

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this package, and only as the checker or the
CPU baseline.  The product package (paper_2001_07809_b200) never imports it.

Both libraries expose the same numpy-level interface (class ``Oracle``), so a
test can run one check against either.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libstk_ref.so"
REF_SRC = Path("/root/reference/proj")

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_i16p = np.ctypeslib.ndpointer(np.int16, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class OracleParamError(ValueError):
    """The reference would throw stereotk::ParamError here."""


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (and _ref/ when /root/reference is present)."""
    out = subprocess.run(["make", "-C", str(HERE), "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _ensure_port() -> None:
    if not PORT_SO.exists():
        build()


class Oracle:
    """numpy-level view over either library.  ``kind`` is "port" or "reference"."""

    def __init__(self, kind: str):
        self.kind = kind
        if kind == "port":
            _ensure_port()
            self.lib = C.CDLL(str(PORT_SO))
            p = "orc_"
        elif kind == "reference":
            if not REF_SO.exists():
                raise FileNotFoundError(REF_SO)
            self.lib = C.CDLL(str(REF_SO))
            p = "ref_"
        else:
            raise ValueError(kind)
        self._p = p
        L = self.lib
        if kind == "reference":
            L.ref_last_error.restype = C.c_char_p
            L.ref_lightness.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, _u8p]
            L.ref_histogram.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, _u64p]
            L.ref_kmeans.argtypes = [_u64p, C.c_int, C.c_int, C.c_double, _f64p, _u16p,
                                     C.POINTER(C.c_int)]
            L.ref_detect.argtypes = [_u16p, C.c_int, C.c_int, _u8p]
            for f in ("ref_fill", "ref_remove"):
                getattr(L, f).argtypes = [_u8p, C.c_int, C.c_int, _u8p]
            L.ref_label_components.argtypes = [_u8p, C.c_int, C.c_int, _i32p, _u32p, _i32p]
            L.ref_prune.argtypes = [_u8p, C.c_int, C.c_int, C.c_double, _u8p]
            L.ref_anchors.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, _u8p]
            L.ref_match.argtypes = [_u8p, _u8p, _u8p, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_int, _i16p]
            L.ref_fill_scanlines.argtypes = [_i16p, C.c_int, C.c_int, _i16p]
            L.ref_peek_columns.argtypes = [_i16p, C.c_int, C.c_int, C.c_int, _i16p]
            L.ref_gaussian_kernel.argtypes = [C.c_double, C.c_int, _f64p]
            L.ref_blur_map.argtypes = [_i16p, C.c_int, C.c_int, _i32p, _i32p, C.c_int,
                                       C.c_int, _u8p]
            L.ref_selective_blur.argtypes = [_u8p, _u8p, C.c_int, C.c_int, C.c_double,
                                             C.c_int, C.c_int, _u8p]
            L.ref_hardware_workers.restype = C.c_int
            L.ref_dense_sad_baseline.argtypes = [_u8p, _u8p, C.c_int, C.c_int, C.c_int, C.c_int,
                                                 C.c_int, _i16p]
            L.ref_bad_pixel_rate.argtypes = [_i16p, _i16p, C.c_int, C.c_int, C.c_double, C.c_int,
                                             C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                             C.POINTER(C.c_uint64), C.c_char_p, C.c_int]
        else:
            L.orc_lightness.argtypes = [_u8p, C.c_int, C.c_int, _u8p]
            L.orc_histogram.argtypes = [_u8p, C.c_size_t, _u64p]
            L.orc_kmeans.argtypes = [_u64p, C.c_int, C.c_int, C.c_double, _f64p, _u16p,
                                     C.POINTER(C.c_int)]
            L.orc_detect.argtypes = [_u16p, C.c_int, C.c_int, _u8p]
            for f in ("orc_fill", "orc_remove"):
                getattr(L, f).argtypes = [_u8p, C.c_int, C.c_int, _u8p]
            L.orc_label_components.argtypes = [_u8p, C.c_int, C.c_int, _i32p, _u32p, _i32p]
            L.orc_prune.argtypes = [_u8p, C.c_int, C.c_int, C.c_double, _u8p]
            L.orc_anchors.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, _u8p]
            L.orc_sad_cost.argtypes = [_u8p, _u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
            L.orc_sad_cost.restype = C.c_uint32
            L.orc_match.argtypes = [_u8p, _u8p, _u8p, C.c_int, C.c_int, C.c_int, C.c_int, _i16p]
            L.orc_fill_scanlines.argtypes = [_i16p, C.c_int, C.c_int, _i16p]
            L.orc_peek_columns.argtypes = [_i16p, C.c_int, C.c_int, C.c_int, _i16p]
            L.orc_default_kernel_size.argtypes = [C.c_double]
            L.orc_gaussian_kernel.argtypes = [C.c_double, C.c_int, _f64p]
            L.orc_blur_map.argtypes = [_i16p, C.c_int, C.c_int, _i32p, _i32p, C.c_int,
                                       C.c_int, _u8p]
            L.orc_selective_blur.argtypes = [_u8p, _u8p, C.c_int, C.c_int, _f64p, C.c_int, _u8p]
            for f in ("orc_lightness", "orc_histogram", "orc_detect", "orc_fill", "orc_remove",
                      "orc_fill_scanlines", "orc_selective_blur"):
                getattr(L, f).restype = None

    # ------------------------------------------------------------ helpers --
    def _check(self, rc):
        if rc < 0:
            msg = self.lib.ref_last_error().decode() if self.kind == "reference" else "param"
            raise OracleParamError(msg)
        return rc

    # ------------------------------------------------------------- stages --
    def lightness(self, rgb: np.ndarray, workers: int = 1) -> np.ndarray:
        h, w = rgb.shape[:2]
        rgb = np.ascontiguousarray(rgb, np.uint8)
        out = np.empty((h, w), np.uint8)
        if self.kind == "reference":
            self._check(self.lib.ref_lightness(rgb.reshape(-1), w, h, workers, out.reshape(-1)))
        else:
            self.lib.orc_lightness(rgb.reshape(-1), w, h, out.reshape(-1))
        return out

    def histogram(self, gray: np.ndarray) -> np.ndarray:
        gray = np.ascontiguousarray(gray, np.uint8)
        out = np.zeros(256, np.uint64)
        if self.kind == "reference":
            h, w = gray.shape
            self._check(self.lib.ref_histogram(gray.reshape(-1), w, h, 1, out))
        else:
            self.lib.orc_histogram(gray.reshape(-1), gray.size, out)
        return out

    def kmeans(self, counts, k, max_iter=100, tol=0.5):
        counts = np.ascontiguousarray(counts, np.uint64)
        centers = np.zeros(max(k, 1), np.float64)
        asg = np.zeros(256, np.uint16)
        it = C.c_int(0)
        fn = self.lib.ref_kmeans if self.kind == "reference" else self.lib.orc_kmeans
        self._check(fn(counts, k, max_iter, tol, centers, asg, C.byref(it)))
        return centers[:k].copy(), asg, it.value

    def detect(self, labels: np.ndarray) -> np.ndarray:
        labels = np.ascontiguousarray(labels, np.uint16)
        h, w = labels.shape
        out = np.empty((h, w), np.uint8)
        self._check(getattr(self.lib, self._p + "detect")(labels.reshape(-1), w, h, out.reshape(-1)) or 0)
        return out

    def _mask_op(self, name, mask):
        mask = np.ascontiguousarray(mask, np.uint8)
        h, w = mask.shape
        out = np.empty((h, w), np.uint8)
        rc = getattr(self.lib, self._p + name)(mask.reshape(-1), w, h, out.reshape(-1))
        self._check(rc or 0)
        return out

    def fill(self, mask):
        return self._mask_op("fill", mask)

    def remove(self, mask):
        return self._mask_op("remove", mask)

    def label_components(self, mask):
        mask = np.ascontiguousarray(mask, np.uint8)
        h, w = mask.shape
        labels = np.empty((h, w), np.int32)
        sizes = np.zeros(w * h + 1, np.uint32)
        bys = np.zeros(w * h + 1, np.int32)
        n = self._check(getattr(self.lib, self._p + "label_components")(
            mask.reshape(-1), w, h, labels.reshape(-1), sizes, bys))
        return labels, sizes[:n].copy(), bys[:n].copy()

    def prune(self, mask, fraction):
        mask = np.ascontiguousarray(mask, np.uint8)
        h, w = mask.shape
        out = np.empty((h, w), np.uint8)
        self._check(getattr(self.lib, self._p + "prune")(mask.reshape(-1), w, h, fraction,
                                                         out.reshape(-1)))
        return out

    def anchors(self, mask, margin):
        mask = np.ascontiguousarray(mask, np.uint8)
        h, w = mask.shape
        out = np.empty((h, w), np.uint8)
        self._check(getattr(self.lib, self._p + "anchors")(mask.reshape(-1), w, h, margin,
                                                           out.reshape(-1)))
        return out

    def match(self, left, right, mask, window, max_disparity, workers: int = 1):
        left = np.ascontiguousarray(left, np.uint8)
        right = np.ascontiguousarray(right, np.uint8)
        mask = np.ascontiguousarray(mask, np.uint8)
        h, w = left.shape
        out = np.empty((h, w), np.int16)
        if self.kind == "reference":
            self._check(self.lib.ref_match(left.reshape(-1), right.reshape(-1), mask.reshape(-1),
                                           w, h, window, max_disparity, workers, out.reshape(-1)))
        else:
            self._check(self.lib.orc_match(left.reshape(-1), right.reshape(-1), mask.reshape(-1),
                                           w, h, window, max_disparity, out.reshape(-1)))
        return out

    def dense_sad_baseline(self, left, right, window, max_disparity, workers: int = 1):
        """evaluate.cpp:92-135 -- the port restates it as match() with a full mask
        (every pixel with a valid window; test_evaluate.cpp:125-143 asserts the
        equality)."""
        left = np.ascontiguousarray(left, np.uint8)
        right = np.ascontiguousarray(right, np.uint8)
        h, w = left.shape
        if self.kind == "reference":
            out = np.empty((h, w), np.int16)
            self._check(self.lib.ref_dense_sad_baseline(left.reshape(-1), right.reshape(-1), w, h,
                                                        window, max_disparity, workers,
                                                        out.reshape(-1)))
            return out
        return self.match(left, right, np.ones((h, w), np.uint8), window, max_disparity)

    def bad_pixel_rate(self, computed, truth, delta_d, workers: int = 1):
        """evaluate.cpp:17-74 -> (rate, compared, excluded, report json or None)."""
        computed = np.ascontiguousarray(computed, np.int16)
        truth = np.ascontiguousarray(truth, np.int16)
        h, w = computed.shape
        if self.kind == "reference":
            rate, cmp_, exc = C.c_double(), C.c_uint64(), C.c_uint64()
            buf = C.create_string_buffer(512)
            self._check(self.lib.ref_bad_pixel_rate(computed.reshape(-1), truth.reshape(-1), w, h,
                                                     float(delta_d), workers, C.byref(rate),
                                                     C.byref(cmp_), C.byref(exc), buf, 512))
            return rate.value, cmp_.value, exc.value, buf.value.decode()
        if delta_d < 0:
            raise OracleParamError("bad_pixel_rate: delta_d must be >= 0")
        known = (computed >= 0) & (truth >= 0)
        compared = int(known.sum())
        diff = np.abs(computed.astype(np.int32) - truth.astype(np.int32))
        bad = int((known & (diff > delta_d)).sum())
        return (0.0 if compared == 0 else bad / compared), compared, w * h - compared, None

    def sad_cost(self, left, right, x, y, d, window):
        assert self.kind == "port"
        left = np.ascontiguousarray(left, np.uint8)
        right = np.ascontiguousarray(right, np.uint8)
        return self.lib.orc_sad_cost(left.reshape(-1), right.reshape(-1), left.shape[1], x, y,
                                     d, window)

    def fill_scanlines(self, sparse):
        sparse = np.ascontiguousarray(sparse, np.int16)
        h, w = sparse.shape
        out = np.empty((h, w), np.int16)
        rc = getattr(self.lib, self._p + "fill_scanlines")(sparse.reshape(-1), w, h,
                                                           out.reshape(-1))
        self._check(rc or 0)
        return out

    def peek_columns(self, m, threshold):
        m = np.ascontiguousarray(m, np.int16)
        h, w = m.shape
        out = np.empty((h, w), np.int16)
        self._check(getattr(self.lib, self._p + "peek_columns")(m.reshape(-1), w, h, threshold,
                                                                out.reshape(-1)))
        return out

    def gaussian_kernel(self, sigma, size):
        out = np.zeros(max(size, 1) ** 2, np.float64)
        self._check(getattr(self.lib, self._p + "gaussian_kernel")(sigma, size, out))
        return out.reshape(size, size)

    def blur_map(self, depth, ranges, max_disparity):
        depth = np.ascontiguousarray(depth, np.int16)
        h, w = depth.shape
        lo = np.array([r[0] for r in ranges] or [0], np.int32)
        hi = np.array([r[1] for r in ranges] or [0], np.int32)
        out = np.empty((h, w), np.uint8)
        self._check(getattr(self.lib, self._p + "blur_map")(depth.reshape(-1), w, h, lo, hi,
                                                            len(ranges), max_disparity,
                                                            out.reshape(-1)))
        return out

    def selective_blur(self, rgb, blur_map, sigma, size, workers: int = 1):
        rgb = np.ascontiguousarray(rgb, np.uint8)
        blur_map = np.ascontiguousarray(blur_map, np.uint8)
        h, w = blur_map.shape
        out = np.empty_like(rgb)
        if self.kind == "reference":
            self._check(self.lib.ref_selective_blur(rgb.reshape(-1), blur_map.reshape(-1), w, h,
                                                    sigma, size, workers, out.reshape(-1)))
        else:
            wts = self.gaussian_kernel(sigma, size).reshape(-1).copy()
            self.lib.orc_selective_blur(rgb.reshape(-1), blur_map.reshape(-1), w, h, wts, size,
                                        out.reshape(-1))
        return out

    # ----------------------------------------------------- whole pipeline --
    def run_frame(self, left, right, *, k=10, window=9, max_disparity=16, threshold=1,
                  prune_fraction=0.04, focus=None, sigma=2.0, kernel_size=0, workers=1):
        """run_refocus_pipeline (or run_depth_pipeline when focus is None).

        Returns a dict with every DepthResult intermediate, stats, the refocused
        image (if focus) and the per-stage ms (reference kind only)."""
        left = np.ascontiguousarray(left, np.uint8)
        right = np.ascontiguousarray(right, np.uint8)
        h, w = left.shape[:2]
        n = w * h
        res = {
            "left_lightness": np.empty((h, w), np.uint8),
            "right_lightness": np.empty((h, w), np.uint8),
            "labels": np.empty((h, w), np.uint16),
            "boundary_raw": np.empty((h, w), np.uint8),
            "boundary_refined": np.empty((h, w), np.uint8),
            "boundary_anchored": np.empty((h, w), np.uint8),
            "sparse": np.empty((h, w), np.int16),
            "row_filled": np.empty((h, w), np.int16),
            "dense": np.empty((h, w), np.int16),
            "centers": np.zeros(256, np.float64),
            "bin_assignment": np.zeros(256, np.uint16),
        }
        ranges = list(focus or [])
        refocused = np.empty((h, w, 3), np.uint8) if focus else None
        if self.kind == "reference":
            return self._ref_run_frame(left, right, w, h, k, window, max_disparity, threshold,
                                       prune_fraction, workers, ranges, sigma, kernel_size,
                                       refocused, res)
        return self._port_run_frame(left, right, w, h, k, window, max_disparity, threshold,
                                    prune_fraction, ranges, sigma, kernel_size, refocused, res)

    def _ref_run_frame(self, left, right, w, h, k, window, D, thr, frac, workers, ranges, sigma,
                       ksize, refocused, res):
        L = self.lib
        lo = np.array([r[0] for r in ranges] or [0], np.int32)
        hi = np.array([r[1] for r in ranges] or [0], np.int32)
        kit = np.zeros(2, np.int32)
        st = np.zeros(4, np.uint64)
        fr = np.zeros(2, np.float64)
        tm = np.zeros(7, np.float64)

        def P(a):
            return a.ctypes.data_as(C.c_void_p) if a is not None else None

        L.ref_run_frame.restype = C.c_int
        rc = L.ref_run_frame(
            P(left), P(right), C.c_int(w), C.c_int(h), C.c_int(k), C.c_int(window), C.c_int(D),
            C.c_int(thr), C.c_double(frac), C.c_int(workers), P(lo), P(hi), C.c_int(len(ranges)),
            C.c_double(sigma), C.c_int(ksize), P(refocused), P(res["dense"]), P(res["sparse"]),
            P(res["left_lightness"]), P(res["right_lightness"]), P(res["labels"]),
            P(res["boundary_raw"]), P(res["boundary_refined"]), P(res["boundary_anchored"]),
            P(res["row_filled"]), P(res["centers"]), P(res["bin_assignment"]), P(kit), P(st),
            P(fr), P(tm))
        self._check(rc)
        res["k"], res["iterations_run"] = int(kit[0]), int(kit[1])
        res["centers"] = res["centers"][: res["k"]].copy()
        res["stats"] = dict(pixels=int(st[0]), boundary_raw=int(st[1]),
                            boundary_refined=int(st[2]), matched=int(st[3]),
                            matched_fraction=float(fr[0]), known_fraction=float(fr[1]))
        res["times_ms"] = dict(zip(("convert", "segment", "boundary", "match", "fill", "peek",
                                    "blur"), map(float, tm)))
        res["refocused"] = refocused
        return res

    def _port_run_frame(self, left, right, w, h, k, window, D, thr, frac, ranges, sigma, ksize,
                        refocused, res):
        g = {}
        g["l"] = self.lightness(left)
        g["r"] = self.lightness(right)
        hist = self.histogram(g["l"])
        occ = int((hist > 0).sum())
        kk = min(k, occ)
        centers, asg, iters = self.kmeans(hist, kk)
        labels = asg[g["l"]]
        braw = self.detect(labels)
        bref = self.remove(self.fill(braw))
        bref = self.prune(bref, frac)
        banc = self.anchors(bref, window // 2)
        sparse = self.match(g["l"], g["r"], banc, window, D)
        rowf = self.fill_scanlines(sparse)
        dense = self.peek_columns(rowf, thr)
        n = w * h
        res.update(left_lightness=g["l"], right_lightness=g["r"], labels=labels.astype(np.uint16),
                   boundary_raw=braw, boundary_refined=bref, boundary_anchored=banc,
                   sparse=sparse, row_filled=rowf, dense=dense, centers=centers,
                   bin_assignment=asg, k=kk, iterations_run=iters)
        matched = int((sparse >= 0).sum())
        res["stats"] = dict(pixels=n, boundary_raw=int(braw.sum()), boundary_refined=int(bref.sum()),
                            matched=matched, matched_fraction=matched / n if n else 0.0,
                            known_fraction=int((dense >= 0).sum()) / n if n else 0.0)
        if refocused is not None:
            bmap = self.blur_map(dense, ranges, D)
            size = ksize if ksize > 0 else self.lib.orc_default_kernel_size(sigma)
            refocused[...] = self.selective_blur(left, bmap, sigma, size)
        res["refocused"] = refocused
        return res


_cache: dict = {}


def port() -> Oracle:
    if "port" not in _cache:
        _cache["port"] = Oracle("port")
    return _cache["port"]


def reference() -> Oracle | None:
    """The compiled reference, or None when oracle/_ref was not built."""
    if "reference" not in _cache:
        try:
            _cache["reference"] = Oracle("reference")
        except (FileNotFoundError, OSError):
            _cache["reference"] = None
    return _cache["reference"]


def ref_synth(name: str, *args):
    """The reference's own synthetic generators (tests/synthetic.cpp), or None."""
    r = reference()
    if r is None:
        return None
    L = r.lib
    if name in ("bench_frame", "rectangle_scene", "translated_noise"):
        if name == "bench_frame":
            w, h, seed = args
            extra = ()
        else:
            w, h, shift, seed = args
            extra = (C.c_int(shift),)
        l = np.empty((h, w, 3), np.uint8)
        rr = np.empty((h, w, 3), np.uint8)
        getattr(L, "ref_synth_" + name)(C.c_int(w), C.c_int(h), *extra, C.c_uint32(seed),
                                        l.ctypes.data_as(C.c_void_p),
                                        rr.ctypes.data_as(C.c_void_p))
        return l, rr
    if name == "random_rgb":
        w, h, seed = args
        out = np.empty((h, w, 3), np.uint8)
        L.ref_synth_random_rgb(C.c_int(w), C.c_int(h), C.c_uint32(seed), out.ctypes.data_as(C.c_void_p))
        return out
    if name == "random_gray":
        w, h, seed = args
        out = np.empty((h, w), np.uint8)
        L.ref_synth_random_gray(C.c_int(w), C.c_int(h), C.c_uint32(seed), out.ctypes.data_as(C.c_void_p))
        return out
    if name == "random_mask":
        w, h, seed, pct = args
        out = np.empty((h, w), np.uint8)
        L.ref_synth_random_mask(C.c_int(w), C.c_int(h), C.c_uint32(seed), C.c_int(pct),
                                out.ctypes.data_as(C.c_void_p))
        return out
    if name == "random_sparse":
        w, h, seed, pct, dmax = args
        out = np.empty((h, w), np.int16)
        L.ref_synth_random_sparse(C.c_int(w), C.c_int(h), C.c_uint32(seed), C.c_int(pct),
                                  C.c_int(dmax), out.ctypes.data_as(C.c_void_p))
        return out
    raise ValueError(name)


# ------------------------------------------------------------------ file I/O --
class RefIOError(Exception):
    """An exception the reference's file entry points threw: .kind is
    "ParamError" / "IoError" / "FormatError" / "other", .msg its what()."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind, self.msg = kind, msg


_IO_KINDS = {-1: "ParamError", -2: "other", -3: "IoError", -4: "FormatError"}


def _ref_io_call(L, rc):
    if rc != 0:
        raise RefIOError(_IO_KINDS.get(rc, "other"), L.ref_last_error().decode(errors="replace"))


_png_lib: list = []


def ref_png_lib():
    """oracle/_ref/libstk_ref_png.so: the reference library with image_io.cpp
    linked to a real libpng 1.6 (pillow's), or None where it was not built."""
    if not _png_lib:
        so = HERE / "_ref" / "libstk_ref_png.so"
        try:
            _png_lib.append(C.CDLL(str(so)) if so.exists() else None)
        except OSError:
            _png_lib.append(None)
    return _png_lib[0]


def ref_io(name: str, *args, png: bool = False):
    """The reference's own image_io.cpp / evaluate.cpp file entry points
    (compiled against oracle/pngstub/png.h: PGM/PPM only; png=True: the build
    linked to a real libpng, for PNG files).  Raises RefIOError with the
    reference's exception class and message; None without that library."""
    if png:
        L = ref_png_lib()
        if L is None:
            return None
    else:
        r = reference()
        if r is None:
            return None
        L = r.lib
    L.ref_last_error.restype = C.c_char_p
    w, h = C.c_int(), C.c_int()
    if name in ("load_image", "load_gray", "load_disparity", "load_ground_truth"):
        path = str(args[0]).encode()
        if name == "load_image":
            _ref_io_call(L, L.ref_load_image(path, C.byref(w), C.byref(h), None))
            out = np.empty((h.value, w.value, 3), np.uint8)
            _ref_io_call(L, L.ref_load_image(path, C.byref(w), C.byref(h), out.ctypes.data_as(C.c_void_p)))
            return out
        if name == "load_gray":
            _ref_io_call(L, L.ref_load_gray(path, C.byref(w), C.byref(h), None, None, 0))
            out = np.empty((h.value, w.value), np.uint8)
            buf = C.create_string_buffer(1 << 16)
            _ref_io_call(L, L.ref_load_gray(path, C.byref(w), C.byref(h), out.ctypes.data_as(C.c_void_p),
                                            buf, C.c_int(len(buf))))
            return out, buf.value.decode(errors="replace").splitlines()
        fn = L.ref_load_disparity if name == "load_disparity" else L.ref_load_ground_truth
        scale = C.c_double(float(args[1]) if len(args) > 1 else 0.0)
        _ref_io_call(L, fn(path, scale, C.byref(w), C.byref(h), None))
        out = np.empty((h.value, w.value), np.int16)
        _ref_io_call(L, fn(path, scale, C.byref(w), C.byref(h), out.ctypes.data_as(C.c_void_p)))
        return out
    if name == "save_gray":
        img, path = np.ascontiguousarray(args[0], np.uint8), str(args[1]).encode()
        comment = args[2].encode() if len(args) > 2 and args[2] else None
        _ref_io_call(L, L.ref_save_gray(path, img.ctypes.data_as(C.c_void_p), C.c_int(img.shape[1]),
                                        C.c_int(img.shape[0]), comment))
        return None
    if name == "save_rgb":
        img, path = np.ascontiguousarray(args[0], np.uint8), str(args[1]).encode()
        _ref_io_call(L, L.ref_save_rgb(path, img.ctypes.data_as(C.c_void_p), C.c_int(img.shape[1]),
                                       C.c_int(img.shape[0])))
        return None
    if name == "save_disparity":
        d, path = np.ascontiguousarray(args[0], np.int16), str(args[1]).encode()
        _ref_io_call(L, L.ref_save_disparity(path, d.ctypes.data_as(C.c_void_p), C.c_int(d.shape[1]),
                                             C.c_int(d.shape[0]), C.c_double(float(args[2]))))
        return None
    raise ValueError(name)
