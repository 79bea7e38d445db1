export PYTHONPATH=$PWD
OUT=gpurun_out
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e --overlap stacked > $OUT/b15_st_$i.log 2>&1
ZO_PDL=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --overlap stacked > $OUT/b15_stpdl_$i.log 2>&1
ZO_PDL=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > $OUT/b15_nonepdl_$i.log 2>&1
done
