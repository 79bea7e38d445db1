export PYTHONPATH=$PWD
OUT=gpurun_out
mkdir -p $OUT/sanitizer
timeout 300 python tools/sanitize_small.py > $OUT/sanitizer/plain.log 2>&1; echo plain=$? > $OUT/status_g.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_small.py > $OUT/sanitizer/$tool.log 2>&1; echo $tool=$? >> $OUT/status_g.txt
done
