#!/bin/bash
# Round-2 GPU pass (run under gpurun): GPU tests, bench lines, the bench launch list and one
# `ncu --set full` capture per product kernel family (tools/kernel_drivers.py).  Every program
# first exits 0 without ncu, then runs under ncu.  Outputs under $O; summarised into profiles/ by
# tools/ncu_summary.py.
#   bash tools/profile_r02.sh [tag] [parts...]     parts: tests bench launches ncu (default: all)
T=${1:-r02}
shift
PARTS=${*:-tests bench launches ncu}
O=gpurun_out/$T
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
has() { [[ " $PARTS " == *" $1 "* ]]; }
if has tests; then
  timeout 2700 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> $O/pytest_gpu.log
fi
if has bench; then
  timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "exit $?" >> $O/bench_default.log
  for w in config3 config4 csr7 csr_random; do
    timeout 900 python bench.py --workload $w --steps 100 --warmup 10 > $O/bench_$w.log 2>&1
    echo "exit $?" >> $O/bench_$w.log
  done
  timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1
fi
if has launches; then
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
      --log-file $O/launches_config2.csv python bench.py --steps 20 --warmup 20 --no-cpu-baseline --no-schedules --no-tts \
      > $O/ncu_launches_config2.log 2>&1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
      --log-file $O/launches_mg.csv python tools/kernel_drivers.py mg > $O/ncu_launches_mg.log 2>&1
fi
if has ncu; then
  # family | kernel regex | launches to skip | launches to capture
  while IFS='|' read -r fam rx skip cnt; do
    [ -z "$fam" ] && continue
    timeout 600 python tools/kernel_drivers.py $fam > $O/drv_$fam.log 2>&1 || { echo "driver $fam failed" >> $O/drv_$fam.log; continue; }
    timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$rx" -s $skip -c $cnt \
        -o $O/ncu_$fam python tools/kernel_drivers.py $fam > $O/ncu_$fam.log 2>&1
    ncu -i $O/ncu_$fam.ncu-rep --page raw --csv > $O/ncu_$fam.raw.csv 2>/dev/null
    ncu -i $O/ncu_$fam.ncu-rep --page source --print-source cuda,sass --csv > $O/ncu_$fam.source.csv 2>/dev/null
    gzip -f $O/ncu_$fam.source.csv
    # gpurun copies back at most 64 MiB: keep the small reports only
    [ $(stat -c %s $O/ncu_$fam.ncu-rep 2>/dev/null || echo 0) -gt 6000000 ] && rm -f $O/ncu_$fam.ncu-rep
  done <<'EOF'
flood|k_flood_solve_dia|20|1
flood3|k_flood_solve_dia|20|1
sell|k_flood_solve_sell|4|1
sweep|k_flood_dia|1|1
rb|k_rb_half|10|1
seq|k_seq_pipe|0|1
levels|k_level_csr|4|2
frozen|k_lambda|2|2
frozen2|k_corr|1|2
mg|k_restrict|0|1
mg2|k_prolong_add|0|1
mg3|k_rb_mean_half|0|1
mg4|k_residual_dia|0|1
mg5|k_gemv_rows|0|1
mggs|k_gs_rb_half|0|1
line|k_line_mean|0|2
linesolve|k_line_full|0|2
build|k_dia_|0|2
EOF
fi
# stay under gpurun's 64 MiB copy-back limit
while [ $(du -sb gpurun_out | cut -f1) -gt 60000000 ]; do
  f=$(ls -S $O/*.ncu-rep 2>/dev/null | head -1); [ -z "$f" ] && break; rm -f "$f"
done
du -sh $O
tail -3 $O/pytest_gpu.log 2>/dev/null
for f in $O/bench_*.log; do echo "== $f"; tail -c 600 $f; echo; done
echo done > $O/DONE
