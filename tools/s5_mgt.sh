for v in new new2 new new2; do
cp tools/_ab/lib_$v.so paper_1904_04093_b200/libgabp_b200.so
echo lib $v
PROF_MG_TIME=291 python tools/prof_mg.py --J 12 --sigma 2 --cycles 3 2>&1 | tail -1
PROF_MG_TIME=291 python tools/prof_mg.py --J 12 --sigma 2 --cycles 3 --smoother gs 2>&1 | tail -1
done
python -m pytest tests/test_gpu_mg.py tests/test_gpu_configs.py tests/test_line.py -m gpu -x -q 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s5_mg_launches3.csv python tools/prof_mg.py --J 12 --sigma 2 --cycles 4 > gpurun_out/s5_mgl_ncu.log 2>&1
