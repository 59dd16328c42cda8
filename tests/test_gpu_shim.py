"""The C++ drop-in: a program written against the reference's stereotk
headers compiles unchanged against include/stereotk/, links libstk_b200.so,
passes restated reference checks on the B200, and produces the same bytes as
the golden (compiled-reference) frame."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_dropin(tmp_path, golden, port, synth):
    exe = str(tmp_path / "shim_test")
    lib = os.path.join(ROOT, "paper_2001_07809_b200")
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_test.cpp"), "-L", lib, "-lstk_b200",
                    f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    dump = str(tmp_path / "frame.bin")
    r = subprocess.run([exe, dump], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    raw = open(dump, "rb").read()
    n = 96 * 72
    dense = np.frombuffer(raw[: 2 * n], np.int16).reshape(72, 96)
    refoc = np.frombuffer(raw[2 * n: 5 * n], np.uint8).reshape(72, 96, 3)
    boxed = np.frombuffer(raw[5 * n: 8 * n], np.uint8).reshape(72, 96, 3)
    assert (dense == golden["pipe_rect_dense"]).all()
    assert np.abs(refoc.astype(int) - golden["pipe_rect_refocused"].astype(int)).max() <= 1
    # box kernel: exact 2-D path == the oracle's FP64 2-D blur with those weights
    l, _ = synth.rectangle_scene_pair(96, 72, 4, 64)
    w = np.full(9, 1.0 / 9.0)
    want = np.empty_like(l)
    port.lib.orc_selective_blur(l.reshape(-1), np.ones(n, np.uint8), 96, 72, w, 3, want.reshape(-1))
    assert (boxed == want).all()


def test_cpp_run_benchmark_gpus(tmp_path):
    """run_benchmark_gpus: G = 1, 2, 3 contexts (sharing device 0 on a one-GPU
    box), frame f -> GPU f mod G, byte-identical outputs, the CSV layout."""
    exe = str(tmp_path / "bench_gpus_test")
    lib = os.path.join(ROOT, "paper_2001_07809_b200")
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "bench_gpus_test.cpp"), "-L", lib, "-lstk_b200",
                    f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    rows = [l.split(",") for l in r.stdout.strip().split("\n")[1:]]
    assert [x[2] for x in rows[:8]] == ["convert", "segment", "boundary", "match", "fill", "peek",
                                        "blur", "total"]
    assert {x[1] for x in rows} == {"1", "2", "3"}
