OUT=gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/probe tools/sm_probe.cu && /tmp/probe > $OUT/n_probe.txt 2>&1
