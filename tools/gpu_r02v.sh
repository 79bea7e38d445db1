export PYTHONPATH=$PWD
OUT=gpurun_out
rm -f $OUT/v_*
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/v_pytest.log 2>&1; echo pytest=$? > $OUT/status_v.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --offload off --no-cpu-baseline > $OUT/v_bench2.log 2>&1; echo bench2=$? >> $OUT/status_v.txt
echo done >> $OUT/status_v.txt
