set -x
(time python -m pytest tests -m gpu -x -q) > gpurun_out/s5_gputest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5_smoke.log 2>&1
(time python bench.py --steps 20 --warmup 5) > gpurun_out/s5_bench.log 2>&1
(time python bench.py --impl reference --steps 20 --warmup 5) > gpurun_out/s5_bench_ref.log 2>&1
tail -3 gpurun_out/s5_gputest.log; tail -2 gpurun_out/s5_smoke.log; tail -5 gpurun_out/s5_bench.log; tail -5 gpurun_out/s5_bench_ref.log
