O=gpurun_out/r02d; mkdir -p $O
for v in "BGABP_PIPE_PUB=8" "BGABP_PIPE_PUB=4" "BGABP_PIPE_PUB=16" "BGABP_PIPE_PUB=32" "BGABP_PIPE_GATE=24" "BGABP_PIPE_NOUNI=1"; do
  echo "== $v" >> $O/seq_probe.log; env $v SEQ_K=256 timeout 300 python tools/seq_pipe_probe.py >> $O/seq_probe.log 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_seq_pipe -c 1 -o $O/ncu_seq python tools/kernel_drivers.py seq > $O/ncu_seq.log 2>&1
ncu -i $O/ncu_seq.ncu-rep --page raw --csv > $O/ncu_seq.raw.csv 2>/dev/null
ncu -i $O/ncu_seq.ncu-rep --page source --print-source cuda,sass --csv > $O/ncu_seq.source.csv 2>/dev/null; gzip -f $O/ncu_seq.source.csv
rm -f $O/ncu_seq.ncu-rep
cat $O/seq_probe.log
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_gabp.py tests/test_gpu_configs.py tests/test_gpu_sell.py tests/test_gpu_damping.py > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for i in 1 2; do for v in 1 0; do
  BGABP_PDL=$v timeout 300 python bench.py --steps 500 --warmup 20 --no-cpu-baseline --no-schedules --no-tts > $O/bench_pdl$v.$i.log 2>&1
  python -c "import json,sys;d=json.loads([l for l in open('$O/bench_pdl$v.$i.log') if l.startswith('{')][-1]);print('PDL=$v', d['ms_per_step'], d['e2e']['value']/1e9, d['roofline']['us_per_launch'])"
  BGABP_PDL=$v timeout 300 python bench.py --workload config3 --steps 500 --warmup 20 --no-cpu-baseline > $O/bench3_pdl$v.$i.log 2>&1
  python -c "import json,sys;d=json.loads([l for l in open('$O/bench3_pdl$v.$i.log') if l.startswith('{')][-1]);print('config3 PDL=$v', d['ms_per_step'], d['e2e']['value']/1e9, d['roofline']['us_per_launch'], d['solve']['seconds'])"
done; done
BGABP_TIMING=1 timeout 300 python tools/mg_setup_probe.py > $O/mg_setup.log 2>&1; tail -40 $O/mg_setup.log
