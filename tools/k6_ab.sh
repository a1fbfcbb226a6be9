#!/bin/bash
# K6 A/B on one B200 (run under gpurun): bit-exactness of the factors, setup timings of c5 / c4,
# then a -DMHDP_K6_PROF build of k6_patch_lu.cu (cycles per phase) on c5.
set -u
mkdir -p gpurun_out
T=${1:-k6cm}
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_edge.py -q -x -k "patch_lu or sweep_bitexact or singular or large_patches" > gpurun_out/${T}_tests.log 2>&1
timeout 600 python tools/setup_profile.py c5 > gpurun_out/${T}_c5.json 2> gpurun_out/${T}_c5.err
timeout 600 python tools/setup_profile.py c4 > gpurun_out/${T}_c4.json 2> gpurun_out/${T}_c4.err
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fopenmp -DMHDP_K6_PROF \
    -c paper_2104_14855_b200/csrc/k6_patch_lu.cu -o build/k6_patch_lu.cu.o && \
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2104_14855_b200/libmhdp.so build/*.o -Xcompiler -fopenmp -lgomp && \
timeout 600 python tools/setup_profile.py c5 > gpurun_out/${T}_c5_prof.json 2> gpurun_out/${T}_c5_prof.err
echo done > gpurun_out/${T}_done.txt
