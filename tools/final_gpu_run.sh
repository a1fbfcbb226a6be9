#!/bin/bash
# Round-end evidence on one B200 (run under gpurun): GPU suite, smoke, bench line, the
# bench command's ncu launch list, a full ncu capture of the finest-level K2, the setup
# timings (K6 per level, K7) of c5 / c4 and a full ncu capture of the first K6 launch (c5 level 1).
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/final_suite.log 2>&1
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-solves --no-variants --no-cpu-baseline \
    > gpurun_out/final_bench_plain.json 2> gpurun_out/final_bench_plain.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-solves \
    --no-variants --no-cpu-baseline > gpurun_out/final_launches_run.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_patch_apply_tma -c 1 \
    -o gpurun_out/final_k2_full python bench.py --steps 1 --warmup 3 --no-solves --no-variants \
    --no-cpu-baseline > gpurun_out/final_k2_run.log 2>&1
timeout 600 python tools/setup_profile.py c5 > gpurun_out/final_setup_c5.json 2> gpurun_out/final_setup_c5.err
timeout 600 python tools/setup_profile.py c4 > gpurun_out/final_setup_c4.json 2> gpurun_out/final_setup_c4.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_patch_lu_cm -c 1 \
    -o gpurun_out/final_k6_full python tools/setup_profile.py c5 > gpurun_out/final_k6_run.log 2>&1
echo done > gpurun_out/final_done.txt
