O=gpurun_out/r02i; mkdir -p $O
for v in "BGABP_PIPE_APOLL=0" "BGABP_PIPE_APOLL=0 BGABP_PIPE_UNSAFE_NOFENCE=1" "BGABP_PIPE_APOLL=1 BGABP_PIPE_UNSAFE_NOFENCE=1"; do
  echo "== $v" >> $O/seq_probe.log; env $v SEQ_K=256 timeout 300 python tools/seq_pipe_probe.py >> $O/seq_probe.log 2>&1; done
cat $O/seq_probe.log
