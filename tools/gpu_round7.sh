set -x
export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_r7.log 2>&1; echo t=$? >> $OUT/status7.txt
timeout 200 python tools/perturb_bench.py > $OUT/pert_r7.txt 2>&1
timeout 600 python bench.py > $OUT/bench_r7.log 2>&1; echo bench=$? >> $OUT/status7.txt
