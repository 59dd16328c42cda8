# Refresh profiles/<tag>_* from a scripts/gpu_round.sh run merged into gpurun_out/.
#   bash scripts/make_profiles.sh r02
set -e
tag=${1:-r02}
o=gpurun_out; p=profiles
tail -1 $o/bench.log > $p/${tag}_bench_C.json
tail -1 $o/bench_ref.log > $p/${tag}_bench_reference_C.json
cp $o/launches.csv $p/${tag}_launches_C.csv
python scripts/launches_summary.py $o/launches.csv > $p/${tag}_launches_C_summary.txt
python scripts/ncu_to_json.py $o/prof_C.ncu-rep $p/${tag}_ncu_kernels.json
{
  echo "# ncu --set full --clock-control none --import-source on, one B200, the 13 launches of the second"
  echo "# 4096x2304 G2 frame (scripts/gpu_round.sh: python scripts/prof_frame.py --config C --frames 2)."
  echo "# Per-launch times are cold-cache and serialised; bench.py's CUDA-event stage times are the numbers"
  echo "# reported.  Per-kernel metrics: ${tag}_ncu_kernels.json; launch list: ${tag}_launches_C.csv."
  python scripts/ncu_stalls.py $o/prof_C.ncu-rep
  echo
  echo "# k_sad_ws SASS instruction mix (ncu source page, scripts/sass_hot.py)"
  python scripts/sass_hot.py $o/sad_source.csv
  echo
  echo "# k_sad_ws per-region split (scripts/sass_regions.py; regions end at barriers; per-warp counts"
  echo "# average over all 16 warps of a CTA: 8 vertical + 8 horizontal)"
  python scripts/sass_regions.py $o/sad_source.csv
} > $p/${tag}_ncu_full_C_summary.txt
{
  echo "# kernels launched by the stage-entry parity tests (ncu launch list of"
  echo "# pytest tests/test_gpu_stages.py -k 'detect or morph or components or prune'): the"
  echo "# parity surface runs the frame path's B1 (k_morph_bits stage modes) and run CCL (k_ccl_region,"
  echo "# k_ccl_borders) kernels"
  python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/stage_launches.csv")))
hdr = None; c = collections.Counter()
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr): c[dict(zip(hdr, r))["Kernel Name"].split("(")[0]] += 1
for k, n in c.most_common(): print(f"{n:6d}  {k}")
PY
} > $p/${tag}_stage_entry_kernels.txt
ls -la $p | grep $tag
