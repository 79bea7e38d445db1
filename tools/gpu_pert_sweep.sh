export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/pert_g2.txt
ZO_B200_LIB=$PWD/build/alt/libzo_g2.so timeout 300 python -m pytest tests/test_gpu_step.py -q -x -k "perturb or lazy or teacher or graph" > $OUT/g2_t.log 2>&1; echo g2tests=$? >> $OUT/pert_g2.txt
for lib in build/alt/libzo_g2.so paper_2507_03211_b200/lib/libzo_b200.so; do
  for occ in 4 5 6 8; do
    echo "lib=$lib occ=$occ" >> $OUT/pert_g2.txt
    ZO_B200_LIB=$PWD/$lib ZO_PU_OCC=$occ timeout 200 python tools/perturb_bench.py 2>&1 | head -2 >> $OUT/pert_g2.txt
  done
done
