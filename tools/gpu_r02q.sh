export PYTHONPATH=$PWD
OUT=gpurun_out
rm -rf $OUT/q_*
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"attn_pp_kernel" -s 3 -c 1 \
  -o $OUT/q_attn python tools/attn_bench.py > $OUT/q_ncu.log 2>&1
