"""ctypes binding of the C-ABI in include/stk_b200.h (libstk_b200.so).

The library is built in-tree (``_build.py``); importing this module never
falls back to anything else: a missing .so raises immediately, and every
compute entry needs a B200 (the library refuses to create a context
otherwise).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libstk_b200.so"
SYNTH_PATH = PKG / "libstk_synth.so"

STK_OK, STK_EPARAM, STK_EIO, STK_EFORMAT, STK_ECUDA, STK_EINTERNAL = range(6)


class StkConfig(C.Structure):
    _fields_ = [("k", C.c_int), ("window", C.c_int), ("max_disparity", C.c_int),
                ("threshold", C.c_int), ("prune_fraction", C.c_double), ("workers", C.c_int)]


class StkFocus(C.Structure):
    _fields_ = [("lo", C.POINTER(C.c_int)), ("hi", C.POINTER(C.c_int)), ("n_ranges", C.c_int),
                ("sigma", C.c_double), ("kernel_size", C.c_int), ("exact_blur", C.c_int)]


class StkStats(C.Structure):
    _fields_ = [("pixels", C.c_uint64), ("boundary_raw", C.c_uint64),
                ("boundary_refined", C.c_uint64), ("matched", C.c_uint64),
                ("matched_fraction", C.c_double), ("known_fraction", C.c_double)]


class StkTimes(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("convert", "segment", "boundary", "match", "fill", "peek", "blur")]


class StkFrameInfo(C.Structure):
    _fields_ = [("sad_ops", C.c_uint64), ("components", C.c_uint64), ("k", C.c_int),
                ("iterations_run", C.c_int), ("kernels", C.c_int), ("graph", C.c_int),
                ("captured", C.c_int)]


class StkFrameOut(C.Structure):
    _fields_ = [("refocused", C.c_void_p), ("dense", C.c_void_p),
                ("left_lightness", C.c_void_p), ("right_lightness", C.c_void_p),
                ("centers", C.c_void_p), ("bin_assignment", C.c_void_p), ("labels", C.c_void_p),
                ("boundary_raw", C.c_void_p), ("boundary_refined", C.c_void_p),
                ("boundary_anchored", C.c_void_p), ("sparse", C.c_void_p),
                ("row_filled", C.c_void_p)]


class StkVideoOpts(C.Structure):
    _fields_ = [("slots", C.c_int), ("decode_threads", C.c_int), ("write_threads", C.c_int),
                ("png", C.c_int), ("disparity_scale", C.c_double), ("shard_index", C.c_int),
                ("shard_count", C.c_int)]


class StkVideoReport(C.Structure):
    _fields_ = [("frames", C.c_int), ("frames_total", C.c_int), ("wall_s", C.c_double),
                ("frames_per_s", C.c_double), ("decode_s", C.c_double), ("write_s", C.c_double),
                ("gpu_wait_s", C.c_double), ("matched_fraction", C.c_double)]


# name -> (restype, argtypes); every symbol include/stk_b200.h declares.
VP, I, D, SZ = C.c_void_p, C.c_int, C.c_double, C.c_size_t
SIGNATURES = {
    "stk_abi_version": (I, []),
    "stk_device_count": (I, []),
    "stk_status_string": (C.c_char_p, [I]),
    "stk_last_error": (C.c_char_p, [VP]),
    "stk_create": (I, [I, I, I, I, C.POINTER(VP)]),
    "stk_destroy": (None, [VP]),
    "stk_set_sad_kernel": (I, [VP, I]),
    "stk_set_use_graphs": (I, [VP, I]),
    "stk_host_alloc": (I, [SZ, C.POINTER(VP)]),
    "stk_host_free": (None, [VP]),
    "stk_validate_config": (I, [C.POINTER(StkConfig)]),
    "stk_default_kernel_size": (I, [D]),
    "stk_gaussian_kernel": (I, [D, I, VP]),
    "stk_lstar_tables": (None, [VP, VP]),
    "stk_rgb_to_lightness": (I, [VP, VP, I, I, VP]),
    "stk_build_histogram": (I, [VP, VP, I, I, VP]),
    "stk_kmeans_histogram": (I, [VP, VP, I, I, D, VP, VP, C.POINTER(C.c_int)]),
    "stk_assign_pixels": (I, [VP, VP, I, I, VP, I, VP]),
    "stk_detect_boundaries": (I, [VP, VP, I, I, VP]),
    "stk_morph_fill": (I, [VP, VP, I, I, VP]),
    "stk_morph_remove": (I, [VP, VP, I, I, VP]),
    "stk_label_components": (I, [VP, VP, I, I, VP, VP, VP, SZ, C.POINTER(C.c_int)]),
    "stk_prune_components": (I, [VP, VP, I, I, D, VP]),
    "stk_add_border_anchors": (I, [VP, VP, I, I, I, VP]),
    "stk_sad_cost": (I, [VP, VP, VP, I, I, I, I, I, I, C.POINTER(C.c_uint32)]),
    "stk_match_boundary_pixels": (I, [VP, VP, VP, VP, I, I, I, I, VP]),
    "stk_dense_sad_baseline": (I, [VP, VP, VP, I, I, I, I, VP]),
    "stk_probe_sad_peak": (I, [VP, C.POINTER(C.c_double)]),
    "stk_bad_pixel_rate": (I, [VP, VP, VP, I, I, D, C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                               C.POINTER(C.c_uint64)]),
    "stk_fill_scanlines": (I, [VP, VP, I, I, VP]),
    "stk_peek_columns": (I, [VP, VP, I, I, I, VP]),
    "stk_build_blur_map": (I, [VP, VP, I, I, VP, VP, I, I, VP]),
    "stk_selective_blur": (I, [VP, VP, VP, I, I, D, I, I, VP]),
    "stk_selective_blur_weights": (I, [VP, VP, VP, I, I, VP, I, VP]),
    "stk_run_frame": (I, [VP, VP, VP, I, I, C.POINTER(StkConfig), C.POINTER(StkFocus),
                          C.POINTER(StkFrameOut), C.POINTER(StkStats), C.POINTER(StkTimes)]),
    "stk_frame_submit": (I, [VP, I, VP, VP, I, I, C.POINTER(StkConfig), C.POINTER(StkFocus),
                             C.POINTER(StkFrameOut), I]),
    "stk_frame_submit_device": (I, [VP, I, VP, VP, I, I, C.POINTER(StkConfig),
                                    C.POINTER(StkFocus), VP, VP, I]),
    "stk_frame_wait": (I, [VP, I, C.POINTER(StkStats), C.POINTER(StkTimes),
                           C.POINTER(StkFrameInfo)]),
    "stk_slot_stream": (VP, [VP, I]),
    # file I/O (host only)
    "stk_image_probe": (I, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "stk_load_image": (I, [C.c_char_p, VP, I, I]),
    "stk_load_gray": (I, [C.c_char_p, VP, I, I, C.c_char_p, SZ, C.POINTER(SZ)]),
    "stk_save_gray": (I, [C.c_char_p, VP, I, I, C.c_char_p]),
    "stk_save_rgb": (I, [C.c_char_p, VP, I, I]),
    "stk_save_disparity": (I, [C.c_char_p, VP, I, I, D]),
    "stk_load_disparity": (I, [C.c_char_p, VP, I, I, D]),
    "stk_load_ground_truth": (I, [C.c_char_p, VP, I, I, D]),
    "stk_disparity_mask_path": (I, [C.c_char_p, C.c_char_p, SZ, C.POINTER(SZ)]),
    "stk_video_refocus": (I, [VP, C.c_char_p, C.c_char_p, C.POINTER(StkConfig), C.POINTER(StkFocus),
                              C.POINTER(StkVideoOpts), C.POINTER(StkVideoReport)]),
    "stk_list_frame_pairs": (I, [C.c_char_p, C.c_char_p, SZ, C.POINTER(SZ), C.POINTER(C.c_int)]),
}

_lib = None
_synth = None


def lib() -> C.CDLL:
    """Load libstk_b200.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(the CUDA extension is required; there is no CPU path)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def synth_lib() -> C.CDLL:
    global _synth
    if _synth is None:
        if not SYNTH_PATH.exists():
            raise ImportError(f"{SYNTH_PATH} is missing: run __graft_entry__.build()")
        _synth = C.CDLL(str(SYNTH_PATH))
    return _synth
