set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_edge.py tests/test_gpu_golden.py -q -x > gpurun_out/k6cm16_tests.log 2>&1
timeout 600 python tools/setup_profile.py c5 > gpurun_out/k6cm16_c5.json 2> gpurun_out/k6cm16_c5.err
timeout 600 python tools/setup_profile.py c4 > gpurun_out/k6cm16_c4.json 2> gpurun_out/k6cm16_c4.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/k6cm16_smoke.log 2>&1
echo done > gpurun_out/k6cm16_done.txt
