export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/k_*.log $OUT/k_lines.jsonl
timeout 300 python tools/e2e_gap.py fill > $OUT/k_gap_fill.log 2>&1
for rep in 1 2; do
for l2 in off on; do
  timeout 600 python bench.py --offload off --no-cpu-baseline --no-cpu-full --plan fill --l2 $l2 --steps 20 > $OUT/k_bench_fill_$l2.log 2>&1
  grep '^{' $OUT/k_bench_fill_$l2.log >> $OUT/k_lines.jsonl
done
done
timeout 600 python bench.py --offload off --no-cpu-baseline --no-cpu-full --plan stacked --l2 on --steps 20 > $OUT/k_bench_stacked_on.log 2>&1
grep '^{' $OUT/k_bench_stacked_on.log >> $OUT/k_lines.jsonl
python -c "
import ctypes,sys; sys.path.insert(0,'.')
from paper_2507_03211_b200 import ops; print(ops.l2_info())" > $OUT/k_l2info.log 2>&1
echo done > $OUT/status_k.txt
