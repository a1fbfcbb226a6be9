#!/bin/bash
# -DMHDP_K6_PROF build of k6_patch_lu.cu (cycles per phase and LU timeline) on c5; run under gpurun
set -u
mkdir -p gpurun_out
T=${1:-k6prof}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fopenmp -DMHDP_K6_PROF \
    -c paper_2104_14855_b200/csrc/k6_patch_lu.cu -o build/k6_patch_lu.cu.o && \
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2104_14855_b200/libmhdp.so build/*.o -Xcompiler -fopenmp -lgomp && \
timeout 600 python tools/setup_profile.py c5 > gpurun_out/${T}_c5_prof.json 2> gpurun_out/${T}_c5_prof.err
echo done > gpurun_out/${T}_done.txt
