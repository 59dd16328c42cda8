"""Golden PNG-decoding vectors from the reference's OWN decode_png
(image_io.cpp:110-127: libpng simplified API, PNG_FORMAT_RGB, null
background), compiled into oracle/_ref/libstk_ref_png.so against a REAL
libpng 1.6 (pillow's bundled shared library; oracle/Makefile).  Every PNG
colour type and bit depth, tRNS, gAMA / sRGB chunks, Adam7, odd sizes.

    python tests/golden/make_png_golden.py      # writes tests/golden/png_golden.npz
"""
import os
import struct
import sys
import tempfile
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from test_io_cpu import _encode_png, _png_chunk  # noqa: E402


def cases():
    rng = np.random.default_rng(2001)
    gammas = [None, 45455, 100000, 50000, 220000]
    for ctype, depths in ((0, (1, 2, 4, 8, 16)), (2, (8, 16)), (3, (1, 2, 4, 8)), (4, (8, 16)), (6, (8, 16))):
        for depth in depths:
            for w, h in ((7, 5), (33, 17)):
                ch = {0: 1, 2: 3, 3: 1, 4: 2, 6: 4}[ctype]
                hi = (1 << depth) - 1
                s = rng.integers(0, hi + 1, size=(h, w, ch))
                if ctype in (4, 6):  # alphas at the extremes too
                    a = s[..., -1]
                    a[0, :] = 0
                    a[1, :] = hi
                for g in gammas:
                    for variant in ("plain", "trns", "srgb"):
                        if variant == "trns" and ctype not in (0, 2, 3):
                            continue
                        if variant == "srgb" and g is not None:
                            continue
                        extra = b""
                        if ctype == 3:
                            n = 1 << depth
                            pal = rng.integers(0, 256, size=(n, 3)).astype(np.uint8)
                            extra += _png_chunk(b"PLTE", pal.tobytes())
                        if g is not None:
                            extra = _png_chunk(b"gAMA", struct.pack(">I", g)) + extra
                        if variant == "srgb":
                            extra = _png_chunk(b"sRGB", b"\x00") + extra
                        if variant == "trns":
                            if ctype == 3:
                                extra += _png_chunk(b"tRNS", rng.integers(0, 256, size=min(1 << depth, 7)).astype(np.uint8).tobytes())
                            elif ctype == 0:
                                extra += _png_chunk(b"tRNS", struct.pack(">H", int(s[0, 0, 0])))
                            else:
                                extra += _png_chunk(b"tRNS", struct.pack(">HHH", *[int(v) for v in s[0, 0, :3]]))
                        for inter in (False, True):
                            if inter and (w, h) != (33, 17):
                                continue
                            name = f"c{ctype}_d{depth}_{w}x{h}_g{g}_{variant}_{'i' if inter else 'p'}"
                            yield name, _encode_png(s, ctype, depth, inter, extra)


def main():
    if oracle.ref_png_lib() is None:
        raise SystemExit("oracle/_ref/libstk_ref_png.so is missing: run make -C oracle")
    names, blobs, outs, shapes = [], [], [], []
    with tempfile.TemporaryDirectory() as td:
        for name, data in cases():
            p = os.path.join(td, "x.png")
            open(p, "wb").write(data)
            rgb = oracle.ref_io("load_image", p, png=True)
            names.append(name)
            blobs.append(np.frombuffer(data, np.uint8))
            outs.append(rgb.reshape(-1))
            shapes.append(rgb.shape[:2])
    off_b = np.cumsum([0] + [len(b) for b in blobs])
    off_o = np.cumsum([0] + [len(o) for o in outs])
    np.savez_compressed(os.path.join(HERE, "png_golden.npz"), names=np.array(names),
                        png=np.concatenate(blobs), png_off=off_b, rgb=np.concatenate(outs),
                        rgb_off=off_o, shapes=np.array(shapes, np.int32))
    print(f"{len(names)} PNG cases -> tests/golden/png_golden.npz")


if __name__ == "__main__":
    main()
