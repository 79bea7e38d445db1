export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/coresident2.txt
for lib in paper_2507_03211_b200/lib/libzo_b200.so build/alt/libzo_epi4.so; do
  for c in 1 2; do
    ZO_B200_LIB=$PWD/$lib ZO_PU_BG_CTAS=$c timeout 300 python tools/coresident_probe.py >> $OUT/coresident2.txt 2>&1
  done
done
