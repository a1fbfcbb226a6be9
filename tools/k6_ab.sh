#!/bin/bash
# K6 A/B on one B200 (run under gpurun): bit-exactness of the factors, setup timings of c5 / c4,
# optionally an ncu capture of the first k_patch_lu_cm launch (c5 level 1), then a -DMHDP_K6_PROF
# build (cycles per phase and LU timeline) on c5.  usage: k6_ab.sh TAG [ncu]
set -u
mkdir -p gpurun_out
T=${1:-k6cm}
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_edge.py -q -x -k "patch_lu or sweep_bitexact or singular or large_patches" > gpurun_out/${T}_tests.log 2>&1
timeout 600 python tools/setup_profile.py c5 > gpurun_out/${T}_c5.json 2> gpurun_out/${T}_c5.err
timeout 600 python tools/setup_profile.py c4 > gpurun_out/${T}_c4.json 2> gpurun_out/${T}_c4.err
if [ "${2:-}" = "ncu" ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_patch_lu_cm -c 1 \
    -o gpurun_out/${T}_ncu python tools/setup_profile.py c5 > gpurun_out/${T}_ncu.log 2>&1
fi
bash tools/k6_prof.sh ${T}
