#!/bin/bash
# Round profile capture (run under gpurun): each program first exits 0 without ncu, then ncu.
set -x
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-schedules --no-tts > gpurun_out/prof_bench.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_config2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-schedules --no-tts \
    > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_flood_solve_dia -s 6 -c 1 \
    -o gpurun_out/flood_config2 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-schedules --no-tts > gpurun_out/ncu_flood.log 2>&1
SEQ_K=64 python tools/seq_pipe_one.py > gpurun_out/prof_seq.log 2>&1 || exit 1
SEQ_K=64 ncu --set full --import-source on --clock-control none -k regex:k_seq_pipe -c 1 \
    -o gpurun_out/seqpipe_config2 python tools/seq_pipe_one.py > gpurun_out/ncu_seq.log 2>&1
python tools/line_ncu.py > gpurun_out/prof_line.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_line_phase -s 2 -c 2 \
    -o gpurun_out/line_J9 python tools/line_ncu.py > gpurun_out/ncu_line.log 2>&1
echo done
