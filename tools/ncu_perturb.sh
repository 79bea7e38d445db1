#!/bin/bash
# full ncu capture of the fused update+perturb pass (first timed launch of tools/perturb_bench.py)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:perturb_update_kernel -s 2 -c 1 \
  -o gpurun_out/prof_perturb5 python tools/perturb_bench.py > gpurun_out/ncu_p5.log 2>&1
tail -3 gpurun_out/ncu_p5.log
