set -x
export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/status_a.txt
nvidia-smi -L > $OUT/a_smi.txt 2>&1; free -g >> $OUT/a_smi.txt; nproc >> $OUT/a_smi.txt; df -h /dev/shm >> $OUT/a_smi.txt
timeout 300 python __graft_entry__.py smoke > $OUT/a_smoke.log 2>&1; echo smoke=$? >> $OUT/status_a.txt
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/a_pytest.log 2>&1; echo pytest=$? >> $OUT/status_a.txt
timeout 1200 python bench.py > $OUT/a_bench.log 2>&1; echo bench=$? >> $OUT/status_a.txt
