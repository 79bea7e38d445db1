set -x
export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/statusF.txt
timeout 300 python __graft_entry__.py smoke > $OUT/smokeF.log 2>&1; echo smoke=$? >> $OUT/statusF.txt
timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytestF.log 2>&1; echo pytest=$? >> $OUT/statusF.txt
timeout 600 python bench.py > $OUT/benchF1.log 2>&1; echo bench=$? >> $OUT/statusF.txt
timeout 600 python bench.py --no-cpu-baseline > $OUT/benchF2.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/benchF_ref.log 2>&1; echo ref=$? >> $OUT/statusF.txt
ZO_NVTX=1 timeout 600 ncu --nvtx --nvtx-include "zo_step/" --clock-control none --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --log-file $OUT/step_trafficF.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncuFa.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:perturb_update -s 1 -c 1 -o $OUT/profF_perturb python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncuFp.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tcgen05 -s 60 -c 4 -o $OUT/profF_gemm python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncuFg.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn -s 5 -c 1 -o $OUT/profF_attn python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncuFat.log 2>&1
