"""Generate tests/golden/io_golden.json from the COMPILED REFERENCE
(oracle/_ref: the reference's own image_io.cpp + evaluate.cpp, built against
oracle/pngstub/png.h since libpng is absent).

Run in the container where /root/reference exists:
    make -C oracle && python tests/golden/make_io_golden.py

For every reader case in tests/io_cases.py it records the reference's outcome
(exception class and message with the path replaced by "{path}", or the
decoded shape, SHA-256 of the pixels and the header comments), and for every
writer case the SHA-256 of the bytes the reference writes (the value file and
the sibling mask for save_disparity).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import io_cases  # noqa: E402
import oracle  # noqa: E402

OUT = os.path.join(HERE, "io_golden.json")


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def outcome(fn, path):
    try:
        r = fn()
    except oracle.RefIOError as e:
        return {"kind": e.kind, "msg": e.msg.replace(path, "{path}")}
    if isinstance(r, tuple):  # load_gray -> (pixels, comments)
        return {"kind": "ok", "shape": list(r[0].shape), "sha": sha(r[0].tobytes()), "comments": r[1]}
    return {"kind": "ok", "shape": list(r.shape), "sha": sha(r.tobytes())}


def main():
    if oracle.reference() is None:
        raise SystemExit("oracle/_ref/libstk_ref.so missing: build it with make -C oracle")
    g = {"read": {}, "save_gray": {}, "save_rgb": {}, "save_disparity": {}, "load_disparity": {}}
    with tempfile.TemporaryDirectory() as tmp:
        for name, blob in io_cases.pnm_cases():
            p = os.path.join(tmp, name + ".pnm")
            with open(p, "wb") as f:
                f.write(blob)
            g["read"][name] = {
                "load_image": outcome(lambda: oracle.ref_io("load_image", p), p),
                "load_gray": outcome(lambda: oracle.ref_io("load_gray", p), p),
                "load_ground_truth_16": outcome(lambda: oracle.ref_io("load_ground_truth", p, 16.0), p),
                "load_disparity_fb8": outcome(lambda: oracle.ref_io("load_disparity", p, 8.0), p),
            }
        for name, img, comment in io_cases.gray_inputs():
            p = os.path.join(tmp, name + ".pgm")
            oracle.ref_io("save_gray", img, p, comment)
            g["save_gray"][name] = sha(open(p, "rb").read())
        for name, img in io_cases.rgb_inputs():
            p = os.path.join(tmp, name + ".ppm")
            oracle.ref_io("save_rgb", img, p)
            g["save_rgb"][name] = sha(open(p, "rb").read())
        for name, d, scale in io_cases.disparity_inputs():
            p = os.path.join(tmp, name + ".pgm")
            try:
                oracle.ref_io("save_disparity", d, p, scale)
            except oracle.RefIOError as e:
                g["save_disparity"][name] = {"kind": e.kind, "msg": e.msg.replace(p, "{path}")}
                continue
            m = p[:-4] + ".mask.pgm"
            g["save_disparity"][name] = {"kind": "ok", "values": sha(open(p, "rb").read()),
                                         "mask": sha(open(m, "rb").read())}
            back = oracle.ref_io("load_disparity", p)
            g["load_disparity"][name] = sha(back.tobytes())
            os.remove(m)
            back = oracle.ref_io("load_disparity", p, 999.0)
            g["load_disparity"][name + "_nomask"] = sha(back.tobytes())
    with open(OUT, "w") as f:
        json.dump(g, f, indent=1, sort_keys=True)
    print(f"wrote {OUT}: {len(g['read'])} reader cases")


if __name__ == "__main__":
    main()
