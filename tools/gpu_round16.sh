set -x
export PYTHONPATH=$PWD
OUT=gpurun_out
timeout 300 python __graft_entry__.py smoke > $OUT/smoke16.log 2>&1; echo smoke=$? >> $OUT/status16.txt
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest16.log 2>&1; echo pytest=$? >> $OUT/status16.txt
timeout 600 python bench.py > $OUT/bench16.log 2>&1; echo bench=$? >> $OUT/status16.txt
ZO_NVTX=1 timeout 600 ncu --nvtx --nvtx-include "zo_step/" --clock-control none --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --log-file $OUT/step_traffic16.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu16a.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:perturb_update -s 1 -c 1 -o $OUT/prof16_perturb python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu16p.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tcgen05 -s 60 -c 4 -o $OUT/prof16_gemm python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu16g.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn -s 5 -c 1 -o $OUT/prof16_attn python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu16at.log 2>&1
ls -la $OUT | tail -5
