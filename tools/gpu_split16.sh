# 13B offload (T=2048, B=1) with split16 at equal device budgets (lo planes counted in the budget)
export PYTHONPATH=$PWD
mkdir -p gpurun_out/split16b
for m in offload:budget=60:split16 offload:budget=100:split16 offload:budget=40:split16; do
  timeout 900 python tools/run_config.py $m opt-13b 2048 1 4 > gpurun_out/split16b/$(echo $m | tr ':=' '__').json 2> gpurun_out/split16b/err_$(echo $m | tr ':=' '__').txt
done
for f in gpurun_out/split16b/*.json; do python -c "
import json,sys;d=json.load(open('$f'));print(d['mode'],d['median_step_ms'],d.get('stream_busy_ms'),d.get('pcie_gb_per_step'),d['peak_device_gb'],d['g'])"; done
