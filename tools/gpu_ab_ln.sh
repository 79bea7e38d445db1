# LayerNorm: register-resident (ZO_LN_REREAD=0) vs three-pass re-read kernel, microbench + in-step (alternating)
export PYTHONPATH=$PWD
mkdir -p gpurun_out/ln
for v in lnold lnnew; do ZO_B200_LIB=$PWD/paper_2507_03211_b200/lib/libzo_$v.so timeout 120 python tools/ln_bench.py > gpurun_out/ln/micro_$v.txt 2>&1; done
ZO_B200_LIB=$PWD/paper_2507_03211_b200/lib/libzo_lnnew.so timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "layernorm" 2>&1 | tail -1
for i in 1 2 3; do
  for v in lnold lnnew; do
    ZO_B200_LIB=$PWD/paper_2507_03211_b200/lib/libzo_$v.so timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ln/b_${v}_$i.log 2>&1
  done
done
cat gpurun_out/ln/micro_*.txt
for f in gpurun_out/ln/b_*.log; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);b=d['breakdown_ms_per_step'];print('$f',round(d['ms_per_step'],3),'ln',b['zo_layernorm_fwd_split'],d['clocks']['sm_mhz'])"; done
