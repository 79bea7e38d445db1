#!/bin/bash
export PYTHONPATH=$PWD
timeout 600 ncu --set full --import-source on --clock-control none -k regex:perturb_update -s 2 -c 1 \
  -o gpurun_out/prof_perturb2 python tools/perturb_bench.py > gpurun_out/ncu_p2.log 2>&1
