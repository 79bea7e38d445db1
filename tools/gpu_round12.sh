export PYTHONPATH=$PWD
OUT=gpurun_out
for lib in paper_2507_03211_b200/lib/libzo_b200.so build/alt/libzo_epi4.so; do
  for c in 1 2 3; do
    ZO_B200_LIB=$PWD/$lib ZO_PU_BG_CTAS=$c timeout 300 python tools/coresident_probe.py >> $OUT/coresident.txt 2>&1
  done
done
ZO_B200_LIB=$PWD/build/alt/libzo_epi4.so timeout 300 python tools/gemm_bench.py > $OUT/gemm_epi4.txt 2>&1
