export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cur.json 2> gpurun_out/bench_cur.err
python -c "import json;d=json.loads(open('gpurun_out/bench_cur.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), round(d['value']), round(d['e2e']['value']), d['roofline']['frac'], d['clocks'])"
