#!/bin/bash
# Round-end evidence on one B200 (run under gpurun): GPU suite, smoke, bench line, the
# bench command's ncu launch list, and a full ncu capture of the finest-level K2.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/final_suite.log 2>&1
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-solves --no-variants --no-cpu-baseline \
    > gpurun_out/final_bench_plain.json 2> gpurun_out/final_bench_plain.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
    --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-solves \
    --no-variants --no-cpu-baseline > gpurun_out/final_launches_run.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_patch_apply_tma -c 1 \
    -o gpurun_out/final_k2_full python bench.py --steps 1 --warmup 3 --no-solves --no-variants \
    --no-cpu-baseline > gpurun_out/final_k2_run.log 2>&1
echo done > gpurun_out/final_done.txt
