nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
PROF_MG_TIME=291 python tools/prof_mg.py --J 12 --sigma 2 --cycles 3 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s5_mg_launches5.csv python tools/prof_mg.py --J 12 --sigma 2 --cycles 3 > gpurun_out/s5_mgl_ncu.log 2>&1
PROF_MG_TIME=291 python tools/prof_mg.py --J 12 --sigma 2 --cycles 3 2>&1 | tail -2
