#!/bin/bash
# Session-2 profile capture (run under gpurun).  Each program first exits 0 without ncu, then ncu.
# Outputs under gpurun_out/p2_*; summarised into profiles/ by tools/ncu_summary.py.
set -x
O=gpurun_out
python bench.py --steps 20 --warmup 20 --no-cpu-baseline --no-schedules --no-tts > $O/p2_bench.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file $O/p2_launches_config2.csv python bench.py --steps 20 --warmup 20 --no-cpu-baseline --no-schedules --no-tts \
    > $O/p2_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_flood_solve_dia -s 30 -c 1 \
    -o $O/p2_flood_config2 python bench.py --steps 20 --warmup 20 --no-cpu-baseline --no-schedules --no-tts > $O/p2_ncu_flood.log 2>&1
# red-black colour phase (constant-stencil variant) on config 2
python tools/rb_probe.py > $O/p2_rb.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_rb_half -s 10 -c 1 -o $O/p2_rb_config2 python tools/rb_probe.py \
    > $O/p2_ncu_rb.log 2>&1
# config-5 V(2,2) red-black GaBP cycle launch list (J = 12, sigma 1)
python tools/prof_mg.py --J 12 --sigma 1.0 --cycles 2 > $O/p2_mg.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv \
    --log-file $O/p2_launches_mg_J12.csv python tools/prof_mg.py --J 12 --sigma 1.0 --cycles 2 > $O/p2_ncu_mg.log 2>&1
# device layout build of the config-5 fine level (setup kernels)
BGABP_FLOOD2=1 python tools/flood2_probe.py 2 > $O/p2_flood2.log 2>&1 || exit 1
BGABP_FLOOD2=1 ncu --set full --import-source on --clock-control none -k regex:k_flood2 -s 40 -c 1 -o $O/p2_flood2_config2 \
    python tools/flood2_probe.py 2 > $O/p2_ncu_flood2.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_dia_ -c 10 --csv \
    --log-file $O/p2_launches_build.csv python tools/flood2_probe.py 4 > $O/p2_ncu_build.log 2>&1
echo done
