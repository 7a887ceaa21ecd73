python -m pytest tests/test_gpu_gabp.py tests/test_gpu_mg.py -m gpu -x -q 2>&1 | tail -2
BGABP_TIMING=1 python tools/mg_setup_probe.py 2>&1 | tail -40
bash tools/ncu_one.sh s5 frozen k_lambda 2 2
bash tools/ncu_one.sh s5 frozen2 k_corr 1 2
