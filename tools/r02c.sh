O=gpurun_out/r02c; mkdir -p $O
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_mg.py tests/test_problems.py > $O/pytest_mg.log 2>&1; tail -3 $O/pytest_mg.log
timeout 3000 python bench.py --workload mg --mg-sigmas 2 1 --mg-cpu-J 12 --mg-cpu-smoothers gabp_red_black > $O/bench_mg_cpuJ12.log 2>&1
tail -c 4000 $O/bench_mg_cpuJ12.log
