O=gpurun_out/r02m; mkdir -p $O
BGABP_TIMING=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-schedules > $O/bench_timing.log 2>&1
grep -v "^\[mg\]" $O/bench_timing.log | grep -B2 -A12 "config 3\|validate" | head -80
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 1500 -c 400 --csv \
      --log-file $O/launches_mg_cycles.csv python tools/kernel_drivers.py mg > $O/ncu_launches_mg.log 2>&1
tail -2 $O/ncu_launches_mg.log
