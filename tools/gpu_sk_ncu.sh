export PYTHONPATH=$PWD
mkdir -p gpurun_out/sk
for m in dp sk; do
  ZO_SK_POLICY=tail timeout 300 ncu --set full --clock-control none -k regex:gemm_tcgen05 -s 3 -c 1 -o gpurun_out/sk/o_$m python tools/sk_one.py 4096 2048 2048 $m > gpurun_out/sk/log_$m.txt 2>&1
done
ZO_SK_POLICY=tail timeout 300 python tools/sk_ab.py > gpurun_out/sk/ab_tail.txt 2>&1
timeout 300 python tools/sk_ab.py > gpurun_out/sk/ab_two.txt 2>&1
cat gpurun_out/sk/ab_*.txt
