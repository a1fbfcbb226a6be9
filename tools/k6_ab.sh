#!/bin/bash
# K6 A/B on one B200 (run under gpurun): bit-exactness of the factors, setup timings of c5 / c4,
# an ncu capture of the first k_patch_lu_cm launch (c5 level 1), then a -DMHDP_K6_PROF build
# (cycles per phase) on c5.  usage: k6_ab.sh TAG [extra nvcc defines for the variant builds]
set -u
mkdir -p gpurun_out
T=${1:-k6cm}
shift
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_edge.py -q -x -k "patch_lu or sweep_bitexact or singular or large_patches" > gpurun_out/${T}_tests.log 2>&1
timeout 600 python tools/setup_profile.py c5 > gpurun_out/${T}_c5.json 2> gpurun_out/${T}_c5.err
timeout 600 python tools/setup_profile.py c4 > gpurun_out/${T}_c4.json 2> gpurun_out/${T}_c4.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_patch_lu_cm -c 1 \
    -o gpurun_out/${T}_ncu python tools/setup_profile.py c5 > gpurun_out/${T}_ncu.log 2>&1
relink() {
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fopenmp "$@" \
      -c paper_2104_14855_b200/csrc/k6_patch_lu.cu -o build/k6_patch_lu.cu.o && \
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2104_14855_b200/libmhdp.so build/*.o -Xcompiler -fopenmp -lgomp
}
relink -DMHDP_K6_PROF && timeout 600 python tools/setup_profile.py c5 > gpurun_out/${T}_c5_prof.json 2> gpurun_out/${T}_c5_prof.err
for V in "$@"; do
  relink $V && timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_patch_lu_cm -c 1 \
      -o gpurun_out/${T}_ncu${V} python tools/setup_profile.py c5 > gpurun_out/${T}_ncu${V}.log 2>&1
done
echo done > gpurun_out/${T}_done.txt
