# every workload's bench line (N=1) + the reference arm; JSON lines to gpurun_out/bench_<name>.json
# (round 2: the Strang default with the cpu_baseline, every other line without it)
mkdir -p gpurun_out
for w in "ising2d_32768_strang" "ising2d_32768" "ising2d_32768:0.01" "zgb2d_32768" "zgbdiff2d_32768" "zgbodiff2d_32768" \
         "diff2d_8192" "diff2d_8192:0.1" "ising2d_1024" "ising1d_65536" "ising1d_65536x64" "noninteracting1d_1024x1000"; do
  wl=${w%%:*}; dt=${w#*:}; [ "$dt" = "$w" ] && dt=""
  name=$wl${dt:+_dt$dt}
  extra="--no-cpu-baseline"; [ "$wl" = "ising2d_32768_strang" ] && extra=""
  timeout 400 python bench.py --workload $wl ${dt:+--dt $dt} $extra > gpurun_out/bench_$name.log 2> gpurun_out/bench_$name.err
  echo "$name rc=$?"; tail -1 gpurun_out/bench_$name.log > gpurun_out/bench_$name.json
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.log 2>&1; echo ref rc=$?
tail -1 gpurun_out/bench_reference.log > gpurun_out/bench_reference.json
