set -x
export PYTHONPATH=$PWD
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo smoke=$? >> $OUT/status.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo pytest=$? >> $OUT/status.txt
timeout 600 python bench.py > $OUT/bench_default.log 2>&1; echo bench=$? >> $OUT/status.txt
for ov in blocks background; do timeout 400 python bench.py --overlap $ov --no-cpu-baseline > $OUT/bench_$ov.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1100 --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:perturb_update -s 1 -c 1 -o $OUT/prof_perturb python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_p.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tcgen05 -s 100 -c 4 -o $OUT/prof_gemm python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_g.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn -s 10 -c 1 -o $OUT/prof_attn python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_a.log 2>&1
ls -la $OUT
