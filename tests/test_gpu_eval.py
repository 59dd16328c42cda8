"""evaluation on the GPU (reference: evaluate.cpp,
test_evaluate.cpp): bad_pixel_rate and dense_sad_baseline against the oracle
(pinned to the compiled reference in test_oracle_cpu.py) and the reference's
known-answer cases."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
U = -1


def test_bad_pixel_known_answers(dev, stk):
    # test_evaluate.cpp:38-50
    c = np.array([[5, 5], [7, 2]], np.int16)
    t = np.array([[5, 6], [9, 2]], np.int16)
    r = stk.bad_pixel_rate(c, t, 1.0, device=dev)
    assert r.bad_pixel_rate == 0.25 and r.compared == 4 and r.excluded == 0 and r.delta_d == 1.0
    assert stk.bad_pixel_rate(c, t, 0.0, device=dev).bad_pixel_rate == 0.5
    # :52-59 unknowns excluded
    r = stk.bad_pixel_rate(np.array([[5, U, 7]], np.int16), np.array([[5, 3, U]], np.int16), 1.0,
                           device=dev)
    assert (r.compared, r.excluded, r.bad_pixel_rate) == (1, 2, 0.0)
    # :86-92 empty comparison
    r = stk.bad_pixel_rate(np.full((4, 4), U, np.int16), np.full((4, 4), U, np.int16), 1.0, device=dev)
    assert r.compared == 0 and r.bad_pixel_rate == 0.0
    # :94-99 validation
    with pytest.raises(stk.ParamError):
        stk.bad_pixel_rate(np.zeros((4, 4), np.int16), np.zeros((5, 4), np.int16), 1.0, device=dev)
    with pytest.raises(stk.ParamError):
        stk.bad_pixel_rate(np.zeros((4, 4), np.int16), np.zeros((4, 4), np.int16), -0.5, device=dev)


@pytest.mark.parametrize("w,h,seed,delta", [(16, 12, 50, 1.0), (40, 30, 53, 1.0), (333, 77, 7, 0.0),
                                            (1920, 1080, 8, 2.5), (4096, 2304, 9, 1.0)])
def test_bad_pixel_vs_oracle(dev, stk, port, w, h, seed, delta):
    rng = np.random.default_rng(seed)
    a = rng.integers(-1, 40, (h, w)).astype(np.int16)
    b = np.where(rng.random((h, w)) < 0.7, a + rng.integers(-3, 4, (h, w)), -1).astype(np.int16)
    b[b < -1] = -1
    r = stk.bad_pixel_rate(a, b, delta, device=dev)
    rate, cmp_, exc, _ = port.bad_pixel_rate(a, b, delta)
    assert (r.bad_pixel_rate, r.compared, r.excluded) == (rate, cmp_, exc)
    # symmetric (test_evaluate.cpp:61-68)
    r2 = stk.bad_pixel_rate(b, a, delta, device=dev)
    assert (r2.bad_pixel_rate, r2.compared) == (r.bad_pixel_rate, r.compared)
    js = stk.eval_report_json(r)
    assert js.startswith('{"bad_pixel_rate":') and js.endswith("}")


def test_eval_report_json_matches_reference_format(stk):
    r = stk.EvalResult(0.8597616865261228, 1091, 109, 1.0)
    assert stk.eval_report_json(r) == (
        '{"bad_pixel_rate":0.8597616865261228,"compared":1091,"delta_d":1.0,"excluded":109}')


@pytest.mark.parametrize("w,h,win,D", [(24, 20, 3, 6), (200, 60, 9, 16), (640, 120, 15, 64),
                                       (700, 90, 21, 128), (300, 40, 5, 0), (8, 8, 9, 4)])
def test_dense_sad_baseline_vs_oracle(dev, stk, port, synth, w, h, win, D):
    l = synth.random_gray(w, h, w + h)
    r = np.roll(l, -min(D, 4), axis=1) ^ (synth.random_gray(w, h, 3 * w) & 3)
    out = stk.dense_sad_baseline(l, r, stk.MatchConfig(win, D), device=dev)
    np.testing.assert_array_equal(out, port.dense_sad_baseline(l, r, win, D))
    # == the masked matcher on a full mask (test_evaluate.cpp:125-143)
    full = stk.match_boundary_pixels(l, r, np.ones((h, w), np.uint8), stk.MatchConfig(win, D), device=dev)
    np.testing.assert_array_equal(out, full)


def test_dense_sad_baseline_validation(dev, stk):
    g = np.zeros((10, 10), np.uint8)
    with pytest.raises(stk.ParamError, match="window must be odd"):
        stk.dense_sad_baseline(g, g, stk.MatchConfig(4, 8), device=dev)
    with pytest.raises(stk.ParamError, match="max_disparity"):
        stk.dense_sad_baseline(g, g, stk.MatchConfig(3, -1), device=dev)
    with pytest.raises(stk.ParamError, match="image sizes differ"):
        stk.dense_sad_baseline(g, np.zeros((10, 11), np.uint8), stk.MatchConfig(3, 2), device=dev)


@pytest.mark.gpu
def test_probe_sad_peak_plausible(dev, stk):
    # 148 SMs x 64 lanes/clk x 4 byte-ADs at ~1.9 GHz is ~7e13; accept a wide band
    peak = stk.probe_sad_peak()
    assert 1e12 < peak < 1e15, peak
