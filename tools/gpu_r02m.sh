OUT=gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ln tools/ln_bench.cu && /tmp/ln > $OUT/m_ln_bench.txt 2>&1
/tmp/ln >> $OUT/m_ln_bench.txt 2>&1
