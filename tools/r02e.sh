O=gpurun_out/r02u; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_driver.log 2>&1; tail -c 1500 $O/bench_driver.log
timeout 600 python tools/kernel_drivers.py seq > /dev/null 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_seq_pipe -c 1 -o $O/ncu_seq python tools/kernel_drivers.py seq > $O/ncu_seq.log 2>&1
ncu -i $O/ncu_seq.ncu-rep --page raw --csv > $O/ncu_seq.raw.csv 2>/dev/null; rm -f $O/ncu_seq.ncu-rep
