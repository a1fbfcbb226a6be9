#!/bin/bash
# K7 / PivotDiv check on one B200 (run under gpurun): coarse-solve and K7 bit-exactness, the PivotDiv pin,
# then the setup timings of c5 / c4 / c3.
set -u
mkdir -p gpurun_out
T=${1:-k7}
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_edge.py -q -x > gpurun_out/${T}_tests.log 2>&1
timeout 600 python tools/setup_profile.py c5 > gpurun_out/${T}_c5.json 2> gpurun_out/${T}_c5.err
timeout 600 python tools/setup_profile.py c4 > gpurun_out/${T}_c4.json 2> gpurun_out/${T}_c4.err
timeout 600 python tools/setup_profile.py c3 > gpurun_out/${T}_c3.json 2> gpurun_out/${T}_c3.err
echo done > gpurun_out/${T}_done.txt
