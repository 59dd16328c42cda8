# Build a variant of the package into _ab/<name> (git-excluded scratch) with
# extra nvcc flags, for A/B timing on one GPU call:  scripts/ab_build.sh by20 -DSTK_BLUR_BY=20
name=$1; shift
rm -rf _ab/$name && mkdir -p _ab/$name
cp -r paper_2001_07809_b200 include bench.py oracle scripts __graft_entry__.py _ab/$name/ 2>/dev/null
cp MEASURED_PEAKS.json _ab/$name/ 2>/dev/null
rm -rf _ab/$name/paper_2001_07809_b200/build
(cd _ab/$name && STK_NVCC_EXTRA="$*" python -c "from paper_2001_07809_b200 import _build; _build.build(verbose=False)")
