export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/l_lines.jsonl
for rep in 1 2; do
for sk in none zo_layernorm_fwd_split zo_attn_causal_fwd zo_perturb_update zo_layernorm_fwd_split,zo_attn_causal_fwd; do
  ZO_EXP_SKIP=$sk timeout 600 python bench.py --offload off --no-cpu-baseline --no-cpu-full --no-e2e --steps 30 > $OUT/l_bench.log 2>&1
  echo "{\"skip\": \"$sk\", \"line\": $(grep '^{' $OUT/l_bench.log)}" >> $OUT/l_lines.jsonl
done
done
echo done > $OUT/status_l.txt
