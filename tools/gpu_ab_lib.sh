# A/B of two builds of the library on the bench (alternating runs) + the kernel/step tests on the default build
export PYTHONPATH=$PWD
mkdir -p gpurun_out/ab
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -x -q 2>&1 | tail -3
for i in 1 2 3; do
  for v in nopf b200; do
    ZO_B200_LIB=$PWD/paper_2507_03211_b200/lib/libzo_$v.so timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab/${v}_$i.log 2>&1
  done
done
for f in gpurun_out/ab/*.log; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',round(d['ms_per_step'],3),d['breakdown_ms_per_step']['zo_gemm_bf16_split'],d['gemm_us_by_shape'])"; done
