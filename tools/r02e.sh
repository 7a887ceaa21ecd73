O=gpurun_out/r02j; mkdir -p $O
for v in "X=1" "BGABP_PIPE_NOUNI=1"; do
  echo "== $v" >> $O/seq_probe.log; env $v SEQ_K=256 timeout 300 python tools/seq_pipe_probe.py >> $O/seq_probe.log 2>&1; done
cat $O/seq_probe.log
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_gabp.py tests/test_gpu_mg.py -k "seq or Sequential or sequential or pipe or lexico or ordered" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
