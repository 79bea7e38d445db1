set -x
export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k attention > $OUT/pytest_r6.log 2>&1; echo t=$? >> $OUT/status6.txt
ZO_B200_LIB=$PWD/build/alt/libzo_kv2.so timeout 120 python tools/attn_bench.py > $OUT/attn_kv2.txt 2>&1
timeout 120 python tools/attn_bench.py > $OUT/attn_kv4.txt 2>&1
for occ in 4 5 6; do ZO_PU_OCC=$occ timeout 200 python tools/perturb_bench.py > $OUT/pert_occ$occ.txt 2>&1; done
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_r6.log 2>&1; echo bench=$? >> $OUT/status6.txt
ZO_B200_LIB=$PWD/build/alt/libzo_kv2.so timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_r6_kv2.log 2>&1
