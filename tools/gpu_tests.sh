# run selected GPU tests: bash tools/gpu_tests.sh "<pytest args>"
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1800 python -m pytest $1 -q -x --timeout 900 > gpurun_out/sel_tests.log 2>&1; echo rc=$? >> gpurun_out/sel_tests.log
