#!/bin/bash
export PYTHONPATH=$PWD
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tcgen05_pair -s 21 -c 1 \
  -o gpurun_out/prof_gemm_pair python tools/gemm_bench.py > gpurun_out/ncu_gp.log 2>&1
