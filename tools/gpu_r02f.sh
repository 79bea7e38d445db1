export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/f_pu.txt
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_zo_core.py -q -x > $OUT/f_tests.log 2>&1; echo tests=$? > $OUT/status_f.txt
for rep in 1 2; do
for v in old r2 r6 r8; do echo "== $v" >> $OUT/f_pu.txt; ZO_B200_LIB=$PWD/build/alt/lib_$v.so timeout 300 python tools/perturb_bench.py >> $OUT/f_pu.txt 2>&1; done
echo "== r4 (default)" >> $OUT/f_pu.txt; timeout 300 python tools/perturb_bench.py >> $OUT/f_pu.txt 2>&1
done
for v in old; do ZO_B200_LIB=$PWD/build/alt/lib_$v.so timeout 600 python bench.py --offload off --no-cpu-baseline --no-cpu-full > $OUT/f_bench_$v.log 2>&1; done
timeout 600 python bench.py --offload off --no-cpu-baseline --no-cpu-full > $OUT/f_bench_r4.log 2>&1
