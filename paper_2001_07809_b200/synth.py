"""Deterministic synthetic stereo scenes (host side; libstk_synth.so).

Byte-identical to the reference's generators (tests/synthetic.cpp) and to the
SURVEY's G2 "dead leaves" scene; pinned against the compiled reference in
tests/test_oracle_cpu.py.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import synth_lib


def _vp(a):
    return a.ctypes.data_as(C.c_void_p)


def _pair(fn, w, h, *args):
    l = np.empty((h, w, 3), np.uint8)
    r = np.empty((h, w, 3), np.uint8)
    fn(C.c_int(w), C.c_int(h), *args, _vp(l), _vp(r))
    return l, r


def dead_leaves(w: int, h: int, max_disparity: int, frame: int = 0, seed: int = None):
    """G2: paper-density scene (~18 % matched boundary pixels); seed 2001+frame."""
    s = 2001 + frame if seed is None else seed
    return _pair(synth_lib().stk_synth_dead_leaves, w, h, C.c_int(max_disparity), C.c_uint32(s))


def bench_frame(w: int, h: int, seed: int):
    """G1: the reference's synthetic::bench_frame (synthetic.cpp:106-127)."""
    return _pair(synth_lib().stk_synth_bench_frame, w, h, C.c_uint32(seed))


def rectangle_scene_pair(w: int, h: int, shift: int, seed: int):
    return _pair(synth_lib().stk_synth_rectangle_scene, w, h, C.c_int(shift), C.c_uint32(seed))


def translated_noise_pair(w: int, h: int, shift: int, seed: int):
    return _pair(synth_lib().stk_synth_translated_noise, w, h, C.c_int(shift), C.c_uint32(seed))


def random_rgb(w: int, h: int, seed: int) -> np.ndarray:
    out = np.empty((h, w, 3), np.uint8)
    synth_lib().stk_synth_random_rgb(C.c_int(w), C.c_int(h), C.c_uint32(seed), _vp(out))
    return out


def random_gray(w: int, h: int, seed: int) -> np.ndarray:
    out = np.empty((h, w), np.uint8)
    synth_lib().stk_synth_random_gray(C.c_int(w), C.c_int(h), C.c_uint32(seed), _vp(out))
    return out


def random_mask(w: int, h: int, seed: int, percent: int) -> np.ndarray:
    out = np.empty((h, w), np.uint8)
    synth_lib().stk_synth_random_mask(C.c_int(w), C.c_int(h), C.c_uint32(seed), C.c_int(percent),
                                      _vp(out))
    return out


def random_sparse(w: int, h: int, seed: int, percent: int, d_max: int) -> np.ndarray:
    out = np.empty((h, w), np.int16)
    synth_lib().stk_synth_random_sparse(C.c_int(w), C.c_int(h), C.c_uint32(seed),
                                        C.c_int(percent), C.c_int(d_max), _vp(out))
    return out


def random_labels(w: int, h: int, seed: int, kinds: int) -> np.ndarray:
    """test_boundary.cpp:26-33: labels[i] = rng() % kinds, raw mt19937 draws."""
    out = np.empty((h, w), np.uint16)
    words = np.empty(w * h, np.uint32)
    _raw_words(seed, words)
    out.reshape(-1)[:] = (words % kinds).astype(np.uint16)
    return out


def _raw_words(seed: int, out: np.ndarray) -> None:
    synth_lib().stk_synth_raw_words(C.c_uint32(seed), C.c_size_t(out.size), _vp(out))
