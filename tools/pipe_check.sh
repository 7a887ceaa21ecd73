#!/bin/bash
# Pipelined lexicographic schedule: GPU parity tests + steady-state timing (tools/seq_pipe_probe.py)
O=gpurun_out/${1:-pipe}; mkdir -p $O
timeout 900 python -m pytest -q -p no:cacheprovider tests -m gpu -k "sequential or seq or pipe or lex or mg or schedule" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
for N in 2048 1024; do
  SEQ_N=$N timeout 300 python tools/seq_pipe_probe.py >> $O/probe.log 2>&1
  SEQ_N=$N BGABP_PIPE_NOUNI=1 timeout 300 python tools/seq_pipe_probe.py >> $O/probe.log 2>&1
done
