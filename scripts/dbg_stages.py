"""Scratch: run each C-ABI stage entry in its own process vs the oracle."""
import subprocess, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
STAGES = ["lightness", "histogram", "kmeans", "assign", "detect", "fill", "remove", "label", "prune",
          "anchors", "match", "fillrows", "peek", "blurmap", "blur", "blurx", "frame"]

def run(stage):
    import numpy as np, oracle
    from paper_2001_07809_b200 import stereotk as s, synth
    o = oracle.port()
    l, r = synth.dead_leaves(450, 375, 16, 0)
    ref = o.run_frame(l, r, k=4, window=9, max_disparity=16, focus=[(8, 16)], sigma=2.0)
    gl, gr = ref["left_lightness"], ref["right_lightness"]
    def eq(a, b):
        a = np.asarray(a); b = np.asarray(b)
        return bool(a.shape == b.shape and (a == b).all()), int((a != b).sum()) if a.shape == b.shape else -1
    if stage == "lightness": print(eq(s.rgb_to_lightness(l), gl))
    if stage == "histogram": print(eq(s.build_histogram(gl), o.histogram(gl)))
    if stage == "kmeans":
        c = s.kmeans_histogram(o.histogram(gl), 4); cc, aa, it = o.kmeans(o.histogram(gl), 4)
        print(eq(c.centers, cc), eq(c.bin_assignment, aa), c.iterations_run, it)
    if stage == "assign":
        c = s.kmeans_histogram(o.histogram(gl), 4); print(eq(s.assign_pixels(gl, c), ref["labels"]))
    if stage == "detect": print(eq(s.detect_boundaries(ref["labels"]), ref["boundary_raw"]))
    if stage == "fill": print(eq(s.morph_fill(ref["boundary_raw"]), o.fill(ref["boundary_raw"])))
    if stage == "remove":
        m = o.fill(ref["boundary_raw"]); print(eq(s.morph_remove(m), o.remove(m)))
    if stage == "label":
        m = o.remove(o.fill(ref["boundary_raw"])); t = s.label_components(m); a, b, c = o.label_components(m)
        print(eq(t.labels, a), eq(t.sizes, b), eq(t.by_size, c))
    if stage == "prune":
        m = o.remove(o.fill(ref["boundary_raw"])); print(eq(s.prune_components(m, 0.04), ref["boundary_refined"]))
    if stage == "anchors": print(eq(s.add_border_anchors(ref["boundary_refined"], 4), ref["boundary_anchored"]))
    if stage == "match": print(eq(s.match_boundary_pixels(gl, gr, ref["boundary_anchored"], s.MatchConfig(9, 16)), ref["sparse"]))
    if stage == "fillrows": print(eq(s.fill_scanlines(ref["sparse"]), ref["row_filled"]))
    if stage == "peek": print(eq(s.peek_columns(ref["row_filled"], 1), ref["dense"]))
    if stage == "blurmap": print(eq(s.build_blur_map(ref["dense"], [(8, 16)], 16), o.blur_map(ref["dense"], [(8, 16)], 16)))
    if stage in ("blur", "blurx"):
        bm = o.blur_map(ref["dense"], [(8, 16)], 16)
        g = s.gaussian_kernel(2.0, 13)
        out = s.selective_blur(l, bm, g, sigma=2.0, exact=(stage == "blurx"))
        d = np.abs(out.astype(int) - ref["refocused"].astype(int)); print("maxdiff", d.max(), "n", (d > 0).sum())
    if stage == "frame":
        dd = []
        out = s.run_refocus_pipeline(l, r, s.PipelineConfig(k=4, window=9, max_disparity=16), s.FocusSpec([(8, 16)], 2.0), depth_out=dd)
        d = dd[0]
        for k in ("left_lightness", "labels", "boundary_raw", "boundary_refined", "boundary_anchored", "sparse", "row_filled", "dense"):
            print(k, eq(getattr(d, k), ref[k]))
        print(d.stats, d.info)

if __name__ == "__main__":
    if len(sys.argv) > 1:
        run(sys.argv[1]); sys.exit(0)
    for st in STAGES:
        p = subprocess.run([sys.executable, __file__, st], capture_output=True, text=True, timeout=120)
        tail = (p.stdout + p.stderr).strip().splitlines()[-8:]
        print(f"== {st} rc={p.returncode}\n   " + "\n   ".join(tail), flush=True)

def sad_cross(cfgname, n=3000, seed=0):
    """strip vs list kernels on a full frame + oracle spot checks (scratch)."""
    import numpy as np, oracle, bench
    from paper_2001_07809_b200 import stereotk as s, synth
    W, H, D, win, K, focus, sigma = bench.CONFIGS[cfgname]
    l, r = synth.dead_leaves(W, H, D, 0)
    dev = s.Device(0)
    cfg = s.PipelineConfig(k=K, window=win, max_disparity=D)
    dev.set_sad_kernel("strip"); a = s.run_depth_pipeline(l, r, cfg, device=dev)
    dev.set_sad_kernel("list"); b = s.run_depth_pipeline(l, r, cfg, device=dev)
    print(cfgname, "strip==list sparse", (a.sparse == b.sparse).all(), "dense", (a.dense == b.dense).all(), "matched", a.stats.matched)
    o = oracle.port()
    ys, xs = np.nonzero(a.sparse >= 0)
    rng = np.random.default_rng(seed); idx = rng.choice(len(ys), size=min(n, len(ys)), replace=False)
    bad = 0
    for i in idx:
        y, x = int(ys[i]), int(xs[i]); dl = min(D, x - win // 2)
        costs = [o.sad_cost(a.left_lightness, a.right_lightness, x, y, d, win) for d in range(dl + 1)]
        bad += int(np.argmin(costs)) != int(a.sparse[y, x])
    print(cfgname, "spot-check mismatches", bad, "of", len(idx))
