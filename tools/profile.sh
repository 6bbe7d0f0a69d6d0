# Profiling pass on the GPU box (one GPU): for each workload, the plain bench run first (must exit 0),
# then the ncu launch list of the same command, then one --set full capture of one window launch.
# Usage: bash tools/profile.sh [workload[:dt] ...]   outputs under gpurun_out/ (tag = workload[@dtDT])
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
for spec in ${@:-ising2d_32768_strang ising2d_32768 zgb2d_32768 diff2d_8192 ising2d_32768:0.01}; do
  w=${spec%%:*}; dt=${spec#*:}; [ "$dt" = "$spec" ] && dt=""
  kind=$w; [ -n "$dt" ] && kind="$w@dt$dt"
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 ${dt:+--dt $dt}"
  timeout 300 $CMD --workload $w > gpurun_out/plain_$kind.log 2> gpurun_out/plain_$kind.err; rc=$?
  echo "$w plain rc=$rc"
  [ $rc -ne 0 ] && continue
  timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv \
      --log-file gpurun_out/launches_$kind.csv $CMD --workload $w > /dev/null 2>&1
  echo "$w launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:substep -s 6 -c 1 \
      -o gpurun_out/prof_$kind -f $CMD --workload $w > gpurun_out/ncu_$kind.log 2>&1
  echo "$w full rc=$?"
done
