# per-block compute and PCIe rates at the OPT-66B / OPT-175B block shapes on one GPU
export PYTHONPATH=$PWD
OUT=gpurun_out/big
mkdir -p $OUT
for m in opt-175b/4 opt-66b/4; do
  n=$(echo $m | tr '/' '_')
  timeout 900 python tools/run_config.py resident $m 2048 1 5 > $OUT/resident_$n.json 2> $OUT/resident_$n.err
  timeout 900 python tools/run_config.py offload $m 2048 1 4 > $OUT/offload_$n.json 2> $OUT/offload_$n.err
  timeout 900 python tools/run_config.py offload:split16 $m 2048 1 4 > $OUT/offload_split16_$n.json 2> $OUT/offload_split16_$n.err
done
echo done > $OUT/status.txt
