O=gpurun_out/r02z; mkdir -p $O
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_gabp.py -k "solve or golden" > $O/pytest.log 2>&1; tail -1 $O/pytest.log
for i in 1 2; do for v in 0 1 2 3; do
  BGABP_DIA_TMA_V=$v timeout 300 python bench.py --steps 500 --warmup 20 --no-cpu-baseline --no-schedules --no-tts > $O/b2.log 2>&1
  python -c "import json;d=json.loads([l for l in open('$O/b2.log') if l.startswith('{')][-1]);print('config2 V=$v', round(d['ms_per_step'],5), round(d['roofline']['us_per_launch'],2), round(d['e2e']['value']/1e9,1))"
done; done
for v in 1 2; do BGABP_DIA_TMA_V=$v timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_gabp.py -k "solve or golden" > $O/pytest$v.log 2>&1; tail -1 $O/pytest$v.log; done
