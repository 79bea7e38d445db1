# build_variants.sh NAME "FLAGS" [NAME "FLAGS" ...]: alternative libraries under build/alt/
# (same sources, extra nvcc defines) for on-GPU A/B runs via ZO_B200_LIB; rebuilds the
# normal library at the end
set -e
mkdir -p build/alt
while [ $# -gt 1 ]; do
  ZO_NVCC_EXTRA="$2" python -c "from paper_2507_03211_b200 import build_lib as b; b.build(force=True)"
  cp paper_2507_03211_b200/lib/libzo_b200.so build/alt/lib_$1.so
  shift 2
done
python -c "from paper_2507_03211_b200 import build_lib as b; b.build(force=True)"
