export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_step.py -q -x -k stacked > $OUT/t32.log 2>&1; echo t=$? > $OUT/status32.txt
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e --overlap stacked_bg > $OUT/b32_bg_$i.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --overlap stacked > $OUT/b32_st_$i.log 2>&1
done
timeout 600 python bench.py --no-cpu-baseline --no-e2e --overlap stacked_bg --no-graph > $OUT/b32_bg_eager.log 2>&1
