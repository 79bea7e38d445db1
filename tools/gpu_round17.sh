export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/pert_sweep.txt
for lib in build/alt/libzo_g2.so paper_2507_03211_b200/lib/libzo_b200.so; do
  for occ in 4 5 6 8; do
    for w in 1 2 4; do
    echo "lib=$lib occ=$occ waves=$w" >> $OUT/pert_sweep.txt
    ZO_B200_LIB=$PWD/$lib ZO_PU_OCC=$occ ZO_PU_WAVES=$w timeout 200 python tools/perturb_bench.py 2>&1 | head -2 >> $OUT/pert_sweep.txt
    done
  done
done
