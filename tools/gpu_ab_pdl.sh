# programmatic dependent launch on / off (ZO_PDL), alternating bench runs
export PYTHONPATH=$PWD
mkdir -p gpurun_out/pdl
for i in 1 2 3; do
  for v in 0 1; do ZO_PDL=$v timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/pdl/b_$v_$i.log 2>&1; cp gpurun_out/pdl/b_$v_$i.log gpurun_out/pdl/pdl${v}_$i.log; done
done
for f in gpurun_out/pdl/pdl*.log; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',round(d['ms_per_step'],3),d['clocks']['sm_mhz'])"; done
