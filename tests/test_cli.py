"""The command-line tool: paper_2001_07809_b200/stereotk,
the reference's tools/main.cpp on libstk_b200.so, driven as a subprocess the
way the reference's tests/test_cli.cpp drives its binary.

CPU tests cover everything that fails before a kernel runs (help, usage
errors, config-file errors, I/O errors, parameter validation) plus the JSON
number format against nlohmann itself; the `gpu` tests run the four
subcommands end to end and check their files against the oracle.
"""
from __future__ import annotations

import json
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

CLI = os.path.join(ROOT, "paper_2001_07809_b200", "stereotk")
NLOHMANN = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"


def run_cli(*args, env=None):
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=300, env=env)
    return r.returncode, r.stdout, r.stderr


@pytest.fixture(scope="module")
def scene(tmp_path_factory, stk, synth):
    """test_cli.cpp:57-70: rectangle_scene_pair(96, 72, 4, 70) as PPM files."""
    d = tmp_path_factory.mktemp("scene")
    left, right = synth.rectangle_scene_pair(96, 72, 4, 70)
    stk.save_rgb(left, d / "scene_L.ppm")
    stk.save_rgb(right, d / "scene_R.ppm")
    return d, str(d / "scene_L.ppm"), str(d / "scene_R.ppm"), left, right


# --------------------------------------------------------------- CPU tests --
def test_help_lists_the_four_commands():
    """test_cli.cpp:74-81"""
    rc, out, _ = run_cli("--help")
    assert rc == 0
    for c in ("depth", "refocus", "eval", "bench"):
        assert c in out
    rc, out, _ = run_cli("depth", "--help")
    assert rc == 0 and "--max-disparity" in out


def test_usage_errors_exit_2(scene):
    """test_cli.cpp:125-144: missing flags / files, bad window."""
    d, L, R, *_ = scene
    assert run_cli()[0] == 2
    assert run_cli("nosuch")[0] == 2
    rc, _, err = run_cli("depth", "--left", L)
    assert rc == 2 and "--right is required" in err
    rc, _, err = run_cli("depth", "--left", "no_such_file.ppm", "--right", R, "--out", d / "x.pgm")
    assert rc == 2 and "error" in err
    rc, _, err = run_cli("depth", "--left", L, "--right", R, "--out", d / "y.pgm", "--window", "4")
    assert rc == 2 and "window" in err
    assert run_cli("depth", "--left", L, "--right", R, "--out", d / "y.pgm", "--k", "two")[0] == 2
    assert run_cli("depth", "--left", L, "--right", R, "--out", d / "y.pgm", "--bogus", "1")[0] == 2
    assert run_cli("depth", "--left", L, "--right", R, "--out", d / "y.pgm", "--scale", "0")[0] == 2


def test_mismatched_inputs_report_both_sizes(stk, tmp_path):
    """test_cli.cpp:109-123"""
    stk.save_rgb(np.zeros((48, 32, 3), np.uint8), tmp_path / "narrow.ppm")
    stk.save_rgb(np.zeros((48, 64, 3), np.uint8), tmp_path / "wide.ppm")
    rc, _, err = run_cli("depth", "--left", tmp_path / "wide.ppm", "--right", tmp_path / "narrow.ppm",
                         "--out", tmp_path / "m.pgm")
    assert rc == 2 and "64x48" in err and "32x48" in err


def test_config_file_errors(scene, tmp_path):
    """test_cli.cpp:146-189 (the parts decided before the GPU runs)."""
    d, L, R, *_ = scene
    cfg = tmp_path / "config.json"
    cfg.write_text('{"window": 4, "k": 2}')
    rc, _, err = run_cli("depth", "--left", L, "--right", R, "--out", tmp_path / "bad.pgm", "--config", cfg)
    assert rc == 2 and "window" in err
    cfg.write_text('{"wnidow": 9}')
    rc, _, err = run_cli("depth", "--left", L, "--right", R, "--out", tmp_path / "u.pgm", "--config", cfg)
    assert rc == 2 and "wnidow" in err
    for text in ('{"k": "two"}', "[1, 2]", "{not json", '{"k": 2,}'):
        cfg.write_text(text)
        assert run_cli("depth", "--left", L, "--right", R, "--out", tmp_path / "f.pgm", "--config", cfg)[0] == 2
    assert run_cli("depth", "--left", L, "--right", R, "--out", tmp_path / "f.pgm", "--config",
                   tmp_path / "missing.json")[0] == 2


def test_refocus_rejects_malformed_focus_and_sigma(scene):
    """test_cli.cpp:207-218"""
    d, L, R, *_ = scene
    base = ["refocus", "--left", L, "--right", R, "--out", d / "refocus_err.ppm"]
    for extra in (["--focus", "abc"], ["--focus", "5"], ["--focus", "7:3"],
                  ["--focus", "1:3", "--sigma", "0"], ["--focus", "1:3", "--kernel-size", "4"]):
        assert run_cli(*base, *extra)[0] == 2, extra


def test_eval_validates_numeric_flags(stk, tmp_path):
    """test_cli.cpp:236-250"""
    t = tmp_path / "flag_truth.pgm"
    stk.save_gray(np.zeros((4, 4), np.uint8), t)
    assert run_cli("eval", t, "--truth", t)[0] == 2
    assert run_cli("eval", t, "--truth", t, "--scale", "0")[0] == 2
    assert run_cli("eval", t, "--truth", t, "--scale", "8", "--delta", "-1")[0] == 2


def test_bench_list_and_directory_errors(stk, tmp_path):
    """test_cli.cpp:283-290"""
    (tmp_path / "empty").mkdir()
    assert run_cli("bench", tmp_path / "empty", "--workers", "1")[0] == 2
    assert run_cli("bench", tmp_path / "nodir", "--workers", "1")[0] == 2
    assert run_cli("bench", tmp_path / "empty", "--workers", "1,x")[0] == 2


def test_json_numbers_match_nlohmann(tmp_path):
    """b200::json_number (the CLI's and eval_report_json's number format) vs
    nlohmann::json::dump() itself, over edge values and 60k random doubles:
    the layout is nlohmann's and the value always round-trips; the digits are
    the shortest round-tripping string, which nlohmann's Grisu2 misses by one
    extra digit (or picks another last digit of a 17-digit string) in ~0.1% of
    cases: same parsed double, never longer."""
    if not os.path.exists(os.path.join(NLOHMANN, "json.hpp")):
        pytest.skip("nlohmann header not present")
    src = tmp_path / "jn.cpp"
    src.write_text(r'''
#include <cstdio>
#include <cstring>
#include <random>
#include <json.hpp>
#include "stereotk/stereotk_b200.hpp"
int main() {
    std::vector<double> v = {0.0, 1.0, -1.0, 0.5, 1000.0, 1e15, 1e16, 123456789012345.0, 1e-4, 1e-5,
                             0.1, 0.25, 1.0/3.0, 2.0/3.0, 1e300, 1e-300, 5e-324, 12.5, 99.99, 1e21,
                             0.0001234, 0.00001234, 4.35, 0.19317, 100.0, 1e-3};
    std::mt19937_64 rng(7);
    for (int i = 0; i < 20000; ++i) {
        double x; uint64_t b = rng(); std::memcpy(&x, &b, 8);
        if (std::isfinite(x)) v.push_back(x);
        v.push_back(double(rng() % 1000000) / double(1 + rng() % 1000));
        v.push_back(double(rng() % 100000) * std::pow(10.0, int(rng() % 40) - 20));
    }
    int diff = 0, bad = 0;
    for (double x : v) {
        const std::string a = nlohmann::json(x).dump(), b = stereotk::b200::json_number(x);
        if (a == b) continue;
        ++diff;
        const bool same = nlohmann::json::parse(b).get<double>() == x && b.size() <= a.size();
        if (!same && bad++ < 10) std::printf("%s vs %s\n", a.c_str(), b.c_str());
    }
    std::printf("differ %d, bad %d of %zu\n", diff, bad, v.size());
    return bad != 0 || diff * 1000 > int(v.size()) * 10;
}''')
    exe = tmp_path / "jn"
    r = subprocess.run(["/usr/bin/g++", "-std=c++17", "-O1", "-I", NLOHMANN, "-I", os.path.join(ROOT, "include"),
                        str(src), "-o", str(exe), "-L", os.path.join(ROOT, "paper_2001_07809_b200"),
                        "-lstk_b200", "-Wl,-rpath," + os.path.join(ROOT, "paper_2001_07809_b200")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout


def test_cli_without_gpu_fails_loudly(scene):
    """No CPU fallback: on a box with no usable GPU the depth command exits 1
    with the library's CUDA error (skipped where a GPU exists)."""
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    d, L, R, *_ = scene
    rc, _, err = run_cli("depth", "--left", L, "--right", R, "--out", d / "nogpu.pgm", "--k", "2",
                         "--max-disparity", "8")
    assert rc == 1 and "no CUDA device" in err


# --------------------------------------------------------------- GPU tests --
@pytest.mark.gpu
def test_depth_map_mask_and_stats(scene, stk, port):
    """test_cli.cpp:83-99, plus the written map == the oracle's dense map."""
    d, L, R, left, right = scene
    out = d / "depth_out.pgm"
    rc, so, err = run_cli("depth", "--left", L, "--right", R, "--out", out, "--k", "2", "--max-disparity", "8",
                          "--window", "9")
    assert rc == 0, err
    assert out.exists() and os.path.exists(stk.disparity_mask_path(out))
    s = json.loads(so)
    assert s["width"] == 96 and s["height"] == 72
    assert 0.0 < s["matched_fraction"] < 1.0 and s["known_fraction"] >= s["matched_fraction"]
    assert set(s["times_ms"]) == {"convert", "segment", "boundary", "match", "fill", "peek", "total"}
    want = port.run_frame(left, right, k=2, window=9, max_disparity=8)
    assert np.array_equal(stk.load_disparity(out), want["dense"])
    assert s["matched"] == want["stats"]["matched"]


@pytest.mark.gpu
def test_depth_reproducible_for_any_workers(scene):
    """test_cli.cpp:101-107"""
    d, L, R, *_ = scene
    a, b = d / "repeat_a.pgm", d / "repeat_b.pgm"
    assert run_cli("depth", "--left", L, "--right", R, "--k", "2", "--max-disparity", "8", "--out", a)[0] == 0
    assert run_cli("depth", "--left", L, "--right", R, "--k", "2", "--max-disparity", "8", "--out", b,
                   "--workers", "4")[0] == 0
    assert a.read_bytes() == b.read_bytes()
    assert (d / "repeat_a.mask.pgm").read_bytes() == (d / "repeat_b.mask.pgm").read_bytes()


@pytest.mark.gpu
def test_config_file_fills_unset_flags(scene, tmp_path):
    """test_cli.cpp:146-189"""
    d, L, R, *_ = scene
    cfg = tmp_path / "config.json"
    cfg.write_text('{"window": 4, "k": 2}')
    out = tmp_path / "config_out.pgm"
    rc, _, err = run_cli("depth", "--left", L, "--right", R, "--out", out, "--config", cfg, "--window", "9",
                         "--max-disparity", "8")
    assert rc == 0, err
    flags = tmp_path / "flags_out.pgm"
    assert run_cli("depth", "--left", L, "--right", R, "--out", flags, "--k", "2", "--window", "9",
                   "--max-disparity", "8")[0] == 0
    assert out.read_bytes() == flags.read_bytes()


@pytest.mark.gpu
def test_depth_debug_dir(scene, stk, port):
    """main.cpp:131-158: every intermediate dumped; sparse/dense decode to the oracle's."""
    d, L, R, left, right = scene
    dbg = d / "dbg"
    rc, _, err = run_cli("depth", "--left", L, "--right", R, "--out", d / "dbg.pgm", "--k", "2",
                         "--max-disparity", "8", "--debug-dir", dbg)
    assert rc == 0, err
    names = {"lightness_left.pgm", "lightness_right.pgm", "labels.pgm", "boundary_raw.pgm",
             "boundary_refined.pgm", "boundary_anchored.pgm", "sparse.pgm", "row_filled.pgm", "dense.pgm"}
    assert names <= set(os.listdir(dbg))
    want = port.run_frame(left, right, k=2, window=9, max_disparity=8)
    assert np.array_equal(stk.load_gray(dbg / "lightness_left.pgm"), want["left_lightness"])
    assert np.array_equal(stk.load_gray(dbg / "boundary_anchored.pgm") > 0, want["boundary_anchored"] > 0)
    assert np.array_equal(stk.load_disparity(dbg / "sparse.pgm"), want["sparse"])


@pytest.mark.gpu
def test_refocus_fully_focused_is_identity(stk, synth, tmp_path):
    """test_cli.cpp:191-205"""
    frame = synth.random_rgb(64, 48, 71)
    p = tmp_path / "flat.ppm"
    stk.save_rgb(frame, p)
    out = tmp_path / "flat_out.ppm"
    rc, so, err = run_cli("refocus", "--left", p, "--right", p, "--out", out, "--k", "2", "--window", "1",
                          "--max-disparity", "8", "--focus", "0:8", "--sigma", "2")
    assert rc == 0, err
    assert out.read_bytes() == p.read_bytes()
    j = json.loads(so)
    assert list(j) == ["matched_fraction", "out"] and j["out"] == str(out)


@pytest.mark.gpu
def test_refocus_png_matches_oracle(scene, stk, port, tmp_path):
    d, L, R, left, right = scene
    out = tmp_path / "refocused.png"
    rc, _, err = run_cli("refocus", "--left", L, "--right", R, "--out", out, "--k", "2", "--max-disparity", "8",
                         "--focus", "3:20", "--sigma", "1.5", "--debug-dir", tmp_path / "dbg")
    assert rc == 0, err
    want = port.run_frame(left, right, k=2, window=9, max_disparity=8, focus=[(3, 8)], sigma=1.5)
    got = stk.load_image(out)
    assert np.abs(got.astype(int) - want["refocused"].astype(int)).max() <= 1
    assert (tmp_path / "dbg" / "blur_map.pgm").exists()


@pytest.mark.gpu
def test_eval_self_is_perfect(stk, tmp_path):
    """test_cli.cpp:220-234"""
    t = np.array([(i % 3) * 8 for i in range(48)], np.uint8).reshape(6, 8)
    p = tmp_path / "self_truth.pgm"
    stk.save_gray(t, p)
    rc, so, err = run_cli("eval", p, "--truth", p, "--scale", "8")
    assert rc == 0, err
    r = json.loads(so)
    assert r == {"bad_pixel_rate": 0.0, "compared": 32, "delta_d": 1.0, "excluded": 16}


@pytest.mark.gpu
def test_bench_csv(stk, synth, tmp_path):
    """test_cli.cpp:252-291"""
    d = tmp_path / "frames"
    d.mkdir()
    for i in range(2):
        l, r = synth.bench_frame(64, 48, 72 + i)
        stk.save_rgb(l, d / f"frame{i}_L.ppm")
        stk.save_rgb(r, d / f"frame{i}_R.ppm")
    rc, so, err = run_cli("bench", d, "--workers", "1", "--max-disparity", "8", "--k", "2")
    assert rc == 0, err
    assert so.startswith("frames,workers,stage,serial_ms,parallel_ms,speedup\n") and ",total," in so
    csv = tmp_path / "bench.csv"
    rc, so, err = run_cli("bench", d, "--workers", "1,2", "--max-disparity", "8", "--k", "2", "--csv", csv)
    assert rc == 0, err
    s = json.loads(so)
    assert csv.exists() and s["frames"] == 2 and len(s["speedup"]) == 2 and s["speedup"]["1"] == 1.0
    assert run_cli("bench", d, "--workers", "2,4")[0] == 2


@pytest.mark.gpu
def test_bench_gpus_csv(stk, synth, tmp_path):
    """stereotk bench --gpus (B200 extension): the GPU-count axis with a blur
    row and GB/s columns; G = 2 runs as two contexts (device g mod count)."""
    d = tmp_path / "frames"
    d.mkdir()
    for i in range(3):
        l, r = synth.dead_leaves(192, 128, 16, frame=i)
        stk.save_rgb(l, d / f"frame{i}_L.ppm")
        stk.save_rgb(r, d / f"frame{i}_R.ppm")
    csv = tmp_path / "gpus.csv"
    rc, so, err = run_cli("bench", d, "--gpus", "1,2", "--max-disparity", "16", "--k", "4",
                          "--focus", "8:16", "--csv", csv)
    assert rc == 0, err
    s = json.loads(so)
    assert s["frames"] == 3 and set(s["speedup"]) == {"1", "2"} and s["speedup"]["1"] == 1.0
    assert set(s["frames_per_s"]) == {"1", "2"} and s["frames_per_s"]["2"] > 0
    text = csv.read_text()
    assert text.startswith("frames,gpus,stage,serial_ms,parallel_ms,speedup,alg_bytes,gb_per_s\n")
    rows = [l.split(",") for l in text.strip().split("\n")[1:]]
    assert len(rows) == 16 and rows[6][2] == "blur" and float(rows[6][4]) > 0
    assert run_cli("bench", d, "--gpus", "2")[0] == 2  # the single-GPU baseline is required
    assert run_cli("bench", d, "--gpus", "1,x")[0] == 2
