export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "embed" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_zo_core.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -3
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'],d['breakdown_ms_per_step'].get('zo_embed_fwd'))"; done
