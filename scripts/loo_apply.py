"""Leave-one-kernel-out experiment: patch a COPY of the package (e.g. _ab/loo,
made by scripts/ab_build.sh-style copying) so that the STK_SKIP bitmask skips
frame-path launches: 1 B1 morph, 2 B2 region, 4 B3 borders, 8 B4 prune,
16 B8 apply, 32 blur, 64 peek, 128 fill, 256 K1, 512 SAD, 1024 K-Means.
Skipping a producer whose output changes the SAD's work (B1, B8, K1,
K-Means) gives meaningless periods.  Usage: python scripts/loo_apply.py ROOT"""
import sys
root = sys.argv[1] + "/paper_2001_07809_b200/csrc/"
edits = {
    "stk_internal.cuh": [("namespace stk {\n", "#include <cstdlib>\nnamespace stk {\n\ninline int skipk(int bit) {\n"
                          "    static const int v = [] { const char* e = getenv(\"STK_SKIP\"); return e ? atoi(e) : 0; }();\n"
                          "    return v & bit;\n}\n")],
    "k_bnd.cu": [("    launch_ccl_region(f, rbits, runroot, bord, st);\n    k_ccl_borders",
                  "    if (!skipk(2)) launch_ccl_region(f, rbits, runroot, bord, st);\n    if (!skipk(4)) k_ccl_borders"),
                 ("        cudaLaunchCooperativeKernel((const void*)k_prune_fused,",
                  "        if (!skipk(8)) cudaLaunchCooperativeKernel((const void*)k_prune_fused,"),
                 ("    k_apply_runs<<<tb, 128, 0, st>>>", "    if (!skipk(16)) k_apply_runs<<<tb, 128, 0, st>>>"),
                 ("    switch (npl) {\n        case 1: k_morph_bits<1, MB_FRAME>",
                  "    if (!skipk(1)) switch (npl) {\n        case 1: k_morph_bits<1, MB_FRAME>")],
    "stk_capi.cu": [("    n += launch_lightness(f, ctx->d_tab, true, true, true, st, ctx->d_lut);",
                     "    if (!skipk(256)) n += launch_lightness(f, ctx->d_tab, true, true, true, st, ctx->d_lut);"),
                    ("    launch_kmeans(f, 0, 100, 0.5, st);", "    if (!skipk(1024)) launch_kmeans(f, 0, 100, 0.5, st);"),
                    ("        launch_sad(f, ctx->sad_kernel, &s.tm_sadL.map, &s.tm_sadR.map, st);\n",
                     "        if (!skipk(512)) launch_sad(f, ctx->sad_kernel, &s.tm_sadL.map, &s.tm_sadR.map, st);\n"),
                    ("    launch_fill_rows(f, f.sparse, f.rowf, st);", "    if (!skipk(128)) launch_fill_rows(f, f.sparse, f.rowf, st);"),
                    ("    launch_peek_cols(f, f.rowf, f.dense, nullptr, st);", "    if (!skipk(64)) launch_peek_cols(f, f.rowf, f.dense, nullptr, st);"),
                    ("    if (bp) n += launch_blur(f, *bp, f.rgbL, f.out_rgb, f.dense, st);",
                     "    if (bp && !skipk(32)) n += launch_blur(f, *bp, f.rgbL, f.out_rgb, f.dense, st);")],
}
for fn, reps in edits.items():
    s = open(root + fn).read()
    for a, b in reps:
        assert a in s, (fn, a[:60])
        s = s.replace(a, b, 1)
    open(root + fn, "w").write(s)
print("patched", root)
