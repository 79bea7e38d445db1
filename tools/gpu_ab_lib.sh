# A/B of two library builds on the bench (alternating runs): ZO_AB="a b" names lib/libzo_<a>.so, lib/libzo_<b>.so
export PYTHONPATH=$PWD
mkdir -p gpurun_out/ab2
for i in 1 2 3; do
  for v in $ZO_AB; do
    ZO_B200_LIB=$PWD/paper_2507_03211_b200/lib/libzo_$v.so timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab2/${v}_$i.log 2>&1
  done
done
for f in gpurun_out/ab2/*.log; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',round(d['ms_per_step'],3),d['breakdown_ms_per_step']['zo_gemm_bf16_split'],{k:v['median_us'] for k,v in d['gemm_us_by_shape'].items()}, d['clocks']['sm_mhz'])"; done
