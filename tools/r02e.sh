O=gpurun_out/r02y; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 20 --no-cpu-baseline --no-schedules --no-tts > $O/b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
      --log-file $O/launches_config2.csv python bench.py --steps 20 --warmup 20 --no-cpu-baseline --no-schedules --no-tts > $O/ncu_launch.log 2>&1
timeout 600 python tools/kernel_drivers.py flood > $O/drv.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_flood_solve_dia -s 20 -c 1 -o $O/ncu_flood python tools/kernel_drivers.py flood > $O/ncu_flood.log 2>&1
ncu -i $O/ncu_flood.ncu-rep --page raw --csv > $O/ncu_flood.raw.csv 2>/dev/null; rm -f $O/ncu_flood.ncu-rep
tail -2 $O/ncu_flood.log
