"""Streamed frame-directory refocus (stk_video_refocus):
decoder threads, GPU slots and writer threads overlapped.  Every output file
must equal run_refocus_pipeline on the same pair (and stay <= 1 LSB of the
oracle); shards partition the frames; a broken frame fails loudly."""
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

W, H, D = 160, 96, 16


@pytest.fixture(scope="module")
def frames_dir(tmp_path_factory, stk, synth):
    d = tmp_path_factory.mktemp("video_in")
    pairs = []
    for f in range(7):
        l, r = synth.dead_leaves(W, H, D, frame=f)
        ext = ".png" if f % 2 else ".ppm"  # mixed formats in one directory
        stk.save_rgb(l, d / f"f{f:03d}_L{ext}")
        stk.save_rgb(r, d / f"f{f:03d}_R{ext}")
        pairs.append((l, r))
    return d, pairs


def _cfg(stk):
    return stk.PipelineConfig(k=4, window=9, max_disparity=D), stk.FocusSpec(ranges=[(8, 16)], sigma=2.0)


@pytest.mark.parametrize("slots,dec,wr,png", [(1, 1, 1, False), (3, 4, 2, False), (2, 3, 1, True)])
def test_video_outputs_equal_single_frame_pipeline(stk, dev, frames_dir, tmp_path, port, slots, dec, wr, png):
    d, pairs = frames_dir
    cfg, focus = _cfg(stk)
    out = tmp_path / "out"
    rep = stk.refocus_video(d, out, cfg, focus, slots=min(slots, dev.slots), decode_threads=dec,
                            write_threads=wr, png=png, disparity_scale=8.0, device=dev)
    assert rep.frames == 7 and rep.frames_total == 7 and rep.frames_per_s > 0
    for f, (l, r) in enumerate(pairs):
        depth = []
        want = stk.run_refocus_pipeline(l, r, cfg, focus, depth_out=depth, device=dev)
        got = stk.load_image(out / (f"f{f:03d}" + (".png" if png else ".ppm")))
        assert np.array_equal(got, want), f
        assert np.array_equal(stk.load_disparity(out / f"f{f:03d}_disp.pgm"), depth[0].dense), f
        if f == 3:
            o = port.run_frame(l, r, k=4, window=9, max_disparity=D, focus=[(8, 16)], sigma=2.0)
            assert np.abs(got.astype(int) - o["refocused"].astype(int)).max() <= 1
            assert np.array_equal(depth[0].dense, o["dense"])


def test_video_shards_partition_frames(stk, dev, frames_dir, tmp_path):
    d, _ = frames_dir
    cfg, focus = _cfg(stk)
    seen = []
    for i in range(3):
        out = tmp_path / f"s{i}"
        rep = stk.refocus_video(d, out, cfg, focus, shard_index=i, shard_count=3, device=dev)
        names = sorted(os.listdir(out))
        assert rep.frames == len(names) and rep.frames_total == 7
        seen += names
    assert sorted(seen) == [f"f{f:03d}.ppm" for f in range(7)]
    with pytest.raises(stk.ParamError):
        stk.refocus_video(d, tmp_path / "bad", cfg, focus, shard_index=3, shard_count=3, device=dev)


def test_video_broken_frame_fails_loudly(stk, dev, frames_dir, tmp_path):
    d, pairs = frames_dir
    bad = tmp_path / "bad_in"
    bad.mkdir()
    for f, (l, r) in enumerate(pairs[:4]):
        stk.save_rgb(l, bad / f"g{f}_L.ppm")
        stk.save_rgb(r, bad / f"g{f}_R.ppm")
    (bad / "g2_R.ppm").write_bytes(b"P6\n160 96\n255\nshort")
    cfg, focus = _cfg(stk)
    with pytest.raises(stk.FormatError, match="truncated"):
        stk.refocus_video(bad, tmp_path / "o", cfg, focus, slots=2, device=dev)
    # the context stays usable afterwards
    l, r = pairs[0]
    assert stk.run_refocus_pipeline(l, r, cfg, focus, device=dev).shape == (H, W, 3)


def test_video_cli(stk, frames_dir, tmp_path):
    d, pairs = frames_dir
    cli = os.path.join(ROOT, "paper_2001_07809_b200", "stereotk")
    out = tmp_path / "cli_out"
    r = subprocess.run([cli, "video", str(d), "--out-dir", str(out), "--focus", "8:16", "--k", "4",
                        "--window", "9", "--max-disparity", str(D), "--slots", "2"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert rep["frames"] == 7 and rep["out_dir"] == str(out)
    cfg, focus = _cfg(stk)
    l, rr = pairs[5]
    assert np.array_equal(stk.load_image(out / "f005.ppm"), stk.run_refocus_pipeline(l, rr, cfg, focus))


def test_video_cli_png_and_disparity(stk, frames_dir, tmp_path, port):
    """`stereotk video --png 1 --disparity-scale 2`: PNG outputs equal the
    pipeline, the disparity files decode to its dense maps."""
    d, pairs = frames_dir
    cli = os.path.join(ROOT, "paper_2001_07809_b200", "stereotk")
    out = tmp_path / "cli_png"
    r = subprocess.run([cli, "video", str(d), "--out-dir", str(out), "--focus", "8:16", "--k", "4",
                        "--window", "9", "--max-disparity", str(D), "--png", "1", "--disparity-scale", "2",
                        "--decode-threads", "3", "--write-threads", "3"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    cfg, focus = _cfg(stk)
    for f in (0, 6):
        l, rr = pairs[f]
        depth = []
        want = stk.run_refocus_pipeline(l, rr, cfg, focus, depth_out=depth)
        assert np.array_equal(stk.load_image(out / f"f{f:03d}.png"), want)
        assert np.array_equal(stk.load_disparity(out / f"f{f:03d}_disp.pgm"), depth[0].dense)
