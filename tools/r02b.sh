O=gpurun_out/r02b; mkdir -p $O
for v in "" "BGABP_PIPE_NOUNI=1" "BGABP_PIPE_MINB=16"; do echo "== $v" >> $O/seq_probe.log; env $v timeout 300 python tools/seq_pipe_probe.py >> $O/seq_probe.log 2>&1; done
timeout 1200 python tools/config5_coarse_rules.py --J 12 --cycles 3000 --sigmas 2 --rules fw_K --no-two-grid > $O/c5_fwK_J12.json 2> $O/c5_fwK_J12.err
timeout 1200 python tools/config5_coarse_rules.py --J 11 --cycles 3000 --sigmas 2 --rules fw_K fw_logK --no-two-grid > $O/c5_fwK_J11.json 2> $O/c5_fwK_J11.err
cat $O/seq_probe.log; tail -c 3000 $O/c5_fwK_J12.json
