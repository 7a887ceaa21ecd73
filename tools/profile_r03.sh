#!/bin/bash
# Final pass of round 2 (run under gpurun): GPU tests, smoke, both bench arms, the bench launch
# list, the multigrid per-cycle launch list and the ncu captures of the kernels touched in the last
# session.  Every program first exits 0 without ncu.  Outputs under gpurun_out/r03.
O=gpurun_out/r03
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 2700 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.log 2>&1; echo "exit $?" >> $O/bench_reference.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_default_20.log 2>&1; echo "exit $?" >> $O/bench_default_20.log
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "exit $?" >> $O/bench_default.log
timeout 900 python bench.py --workload mg --mg-sigmas 2 1 --no-cpu-baseline > $O/bench_mg.log 2>&1; echo "exit $?" >> $O/bench_mg.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_config2.csv python bench.py --steps 20 --warmup 20 --no-cpu-baseline --no-schedules --no-tts \
    > $O/ncu_launches_config2.log 2>&1
python tools/prof_mg.py --J 12 --sigma 2 --cycles 4 > $O/prof_mg.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_mg.csv python tools/prof_mg.py --J 12 --sigma 2 --cycles 4 > $O/ncu_launches_mg.log 2>&1
# the compact-r residual and the phase that reads it (fine level of config 5)
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_residual_dia" -s 0 -c 3 \
    -o $O/ncu_mgres python tools/prof_mg.py --J 12 --sigma 2 --cycles 3 > $O/ncu_mgres.log 2>&1
ncu -i $O/ncu_mgres.ncu-rep --page raw --csv > $O/ncu_mgres.raw.csv 2>/dev/null
# the two launches of a recorded V(2,2) smoothing call (first pair, last pair), fine level
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_rb_mean_(first|last)_pair" -s 0 -c 2 \
    -o $O/ncu_mgphase python tools/prof_mg.py --J 12 --sigma 2 --cycles 3 > $O/ncu_mgphase.log 2>&1
ncu -i $O/ncu_mgphase.ncu-rep --page raw --csv > $O/ncu_mgphase.raw.csv 2>/dev/null
# the phase kernels (V(3,3): the middle sweep runs them)
PROF_MG_SWEEPS=3 python tools/prof_mg.py --J 12 --sigma 2 --cycles 2 > $O/prof_mg_v33.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_rb_mean_half" -s 0 -c 2 \
    -o $O/ncu_mgphase3 env PROF_MG_SWEEPS=3 python tools/prof_mg.py --J 12 --sigma 2 --cycles 2 > $O/ncu_mgphase3.log 2>&1
ncu -i $O/ncu_mgphase3.ncu-rep --page raw --csv > $O/ncu_mgphase3.raw.csv 2>/dev/null
# config 3's nonsymmetric step (out-edge coefficients from the neighbours' row entries)
timeout 900 python bench.py --workload config3 --steps 500 --warmup 20 --no-cpu-baseline > $O/bench_config3.log 2>&1; echo "exit $?" >> $O/bench_config3.log
python tools/kernel_drivers.py flood3 > $O/drv_flood3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_flood_solve_dia" -s 20 -c 1 \
    -o $O/ncu_flood3 python tools/kernel_drivers.py flood3 > $O/ncu_flood3.log 2>&1
ncu -i $O/ncu_flood3.ncu-rep --page raw --csv > $O/ncu_flood3.raw.csv 2>/dev/null
rm -f $O/*.ncu-rep
tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log
for f in $O/bench_*.log; do echo "== $f"; tail -c 400 $f; echo; done
echo done > $O/DONE
