#!/bin/bash
# ncu evidence for profiles/: launch list of a short bench run + full captures
# of the perturb kernel and the largest GEMM.  Run under gpurun (1 GPU).
set -x
export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1100 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:perturb_update -s 1 -c 1 \
  -o $OUT/prof_perturb python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_p.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tcgen05 -s 100 -c 4 \
  -o $OUT/prof_gemm python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_g.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:flash_attn -s 10 -c 1 \
  -o $OUT/prof_attn python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_a.log 2>&1
ls -la $OUT
