"""Deterministic file-format cases shared by tests/test_io_cpu.py and
tests/golden/make_io_golden.py (TEST INFRASTRUCTURE).

PNM_CASES: (name, file bytes) for the reader -- every syntax rule of
image_io.cpp:29-103 (comments between fields, whitespace kinds, exactly one
separator byte, maxval limits, truncation, overflowing fields) plus seeded
random mutations of valid headers.
SAVE_CASES: inputs for the writers (save_gray with/without a comment,
save_rgb to .ppm, save_disparity at several scales incl. overflow/invalid).
"""
from __future__ import annotations

import numpy as np


def _raster(n, seed):
    return np.random.default_rng(seed).integers(0, 256, n, dtype=np.uint8).tobytes()


def pnm_cases():
    c = []
    px6 = _raster(2 * 3 * 3, 1)
    px5 = _raster(4 * 3, 2)
    c += [
        ("p6_basic", b"P6\n2 3\n255\n" + px6),
        ("p5_basic", b"P5\n4 3\n255\n" + px5),
        ("p5_comment_each_field", b"P5\n# a\n4\n#  two spaces\n3 # not a comment here\n255\n" + px5),
        ("p5_comments", b"P5\n# scale 8\n# second\n4 3\n255\n" + px5),
        ("p5_comment_no_space", b"P5\n#scale 8\n4 3\n255\n" + px5),
        ("p5_comment_before_maxval", b"P5 4 3\n# c\n255\n" + px5),
        ("p5_tabs_crlf", b"P5\t4\r\n3\x0b255\n" + px5),
        ("p5_formfeed_sep", b"P5 4 3 255\x0c" + px5),
        ("p5_maxval_15", b"P5 4 3 15\n" + px5),
        ("p5_maxval_256", b"P5 4 3 256\n" + px5),
        ("p5_maxval_0", b"P5 4 3 0\n" + px5),
        ("p5_maxval_65535", b"P5\n1 1\n65535\n\x00\x00"),
        ("p5_zero_width", b"P5 0 3 255\n"),
        ("p5_zero_height", b"P5 4 0 255\n"),
        ("p5_huge_field", b"P5 99999999999 3 255\n"),
        ("p5_field_2pow30", b"P5 1073741824 1 255\n"),
        ("p5_field_2pow30p1", b"P5 1073741825 1 255\n"),
        ("p5_no_separator", b"P5 4 3 255"),
        ("p5_letter_field", b"P5 4 x 255\n" + px5),
        ("p5_negative", b"P5 -4 3 255\n" + px5),
        ("p5_truncated", b"P5 4 3 255\n" + px5[:-1]),
        ("p5_extra_bytes", b"P5 4 3 255\n" + px5 + b"tail"),
        ("p5_two_separators", b"P5 4 3 255\n\n" + px5),
        ("p6_truncated", b"P6\n2 2\n255\nabcde"),
        ("p3_ascii", b"P3\n1 1\n255\n1 2 3\n"),
        ("p2_ascii", b"P2\n1 1\n255\n7\n"),
        ("garbage", b"this is not an image at all\n"),
        ("empty", b""),
        ("one_byte", b"P"),
        ("magic_only", b"P5"),
        ("comment_to_eof", b"P5\n# never ends"),
        ("comment_eof_after_fields", b"P5 4 3 255#x"),
        ("p6_as_gray_source", b"P6 1 1 255\n\x01\x02\x03"),
    ]
    rng = np.random.default_rng(2001)
    base = b"P5\n# c\n5 2\n255\n" + _raster(10, 3)
    alphabet = b"P56 \t\n\r#0123456789x\x0b\x0c"
    for i in range(60):
        b = bytearray(base)
        for _ in range(int(rng.integers(1, 4))):
            pos = int(rng.integers(0, 16))
            op = int(rng.integers(0, 3))
            ch = alphabet[int(rng.integers(0, len(alphabet)))]
            if op == 0 and pos < len(b):
                b[pos] = ch
            elif op == 1:
                b.insert(pos, ch)
            elif pos < len(b):
                del b[pos]
        c.append((f"mutant_{i:02d}", bytes(b)))
    return c


def disparity_inputs():
    rng = np.random.default_rng(7)
    d = rng.integers(-1, 32, (9, 13)).astype(np.int16)
    d[3, 3] = 0
    return [
        ("rand_s8", d, 8.0),
        ("rand_s6", np.clip(d, -1, 42), 6.0),
        ("rand_s0_5", d, 0.5),
        ("rand_s2_25", d, 2.25),
        ("rand_s_third", d, 1.0 / 3.0),
        ("rand_s1e-3", d, 0.001),
        ("rand_s7_999", d, 7.999),
        ("overflow_s8", np.array([[40]], np.int16), 8.0),
        ("ok_s6", np.array([[40]], np.int16), 6.0),
        ("zero_scale", d, 0.0),
        ("neg_scale", d, -2.0),
        ("all_unknown", np.full((4, 5), -1, np.int16), 8.0),
    ]


def gray_inputs():
    rng = np.random.default_rng(11)
    return [
        ("white_1x1", np.array([[255]], np.uint8), None),
        ("seven_nine", np.array([[7, 9]], np.uint8), "scale 8"),
        ("rand_37x21", rng.integers(0, 256, (21, 37), dtype=np.uint8), None),
        ("rand_comment", rng.integers(0, 256, (5, 3), dtype=np.uint8), "any text # with hash"),
    ]


def rgb_inputs():
    rng = np.random.default_rng(12)
    return [
        ("rand_19x33", rng.integers(0, 256, (33, 19, 3), dtype=np.uint8)),
        ("black_1x1", np.zeros((1, 1, 3), np.uint8)),
    ]
