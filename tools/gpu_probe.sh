export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for g in "" "--no-graph"; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline $g > gpurun_out/bench_cur.json 2> gpurun_out/bench_cur.err
python -c "import json;d=json.loads(open('gpurun_out/bench_cur.json').read().strip().splitlines()[-1]);print('$g', round(d['ms_per_step'],3), round(d['value']), round(d['e2e']['value']), d['gpu_launches'], d['clocks'])"
done
