export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k layernorm > $OUT/lnw_tests.log 2>&1; echo tests=$? >> $OUT/lnw_tests.log
timeout 1200 python bench.py --model opt-13b --seq 2048 --batch 1 --steps 10 --offload off --no-cpu-baseline --no-cpu-full > $OUT/lnw_13b.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x --timeout 900 > $OUT/lnw_full.log 2>&1; echo full=$? >> $OUT/lnw_full.log
