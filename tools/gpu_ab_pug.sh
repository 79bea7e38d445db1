# perturb tile width (ZO_PU_G groups per lane) A/B, in-step at 1.3B and 13B, alternating
export PYTHONPATH=$PWD
mkdir -p gpurun_out/pug
for i in 1 2; do
  for v in g4 g8 g2; do
    ZO_B200_LIB=$PWD/paper_2507_03211_b200/lib/libzo_$v.so timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/pug/s_${v}_$i.log 2>&1
    ZO_B200_LIB=$PWD/paper_2507_03211_b200/lib/libzo_$v.so timeout 600 python bench.py --model opt-13b --seq 2048 --batch 1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pug/l_${v}_$i.log 2>&1
  done
done
for f in gpurun_out/pug/*.log; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);b=d['breakdown_ms_per_step'];print('$f',round(d['ms_per_step'],2),'pert',b['zo_perturb_update'],d['clocks']['sm_mhz'])"; done
