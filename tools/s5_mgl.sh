mkdir -p gpurun_out
python tools/prof_mg.py --J 12 --sigma 2 --cycles 4 > gpurun_out/s5_mgl_plain.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s5_mg_launches.csv python tools/prof_mg.py --J 12 --sigma 2 --cycles 4 > gpurun_out/s5_mgl_ncu.log 2>&1
tail -2 gpurun_out/s5_mgl_plain.log; wc -l gpurun_out/s5_mg_launches.csv
