O=gpurun_out/r02t; mkdir -p $O
timeout 1500 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_gabp.py tests/test_gpu_mg.py tests/test_gpu_configs.py tests/test_line.py tests/test_gpu_dropin.py tests/test_cli.py > $O/pytest.log 2>&1; tail -3 $O/pytest.log
SEQ_K=256 timeout 300 python tools/seq_pipe_probe.py
