# A/B on one box: alternate two in-tree builds (A = paper_1105_4673_b200/libkmc_b200_A.so, B = the
# current libkmc_b200.so) over the main workloads, 2 rounds each, short runs
A=paper_1105_4673_b200/libkmc_b200_A.so; B=paper_1105_4673_b200/libkmc_b200.so
for round in 1 2; do
  for lib in A B; do
    path=$A; [ $lib = B ] && path=$B
    for w in ${WORKLOADS:-"ising2d_32768" "ising2d_32768:0.01" "zgb2d_32768" "diff2d_8192"}; do
      wl=${w%%:*}; dt=${w#*:}; [ "$dt" = "$w" ] && dt=""
      KMC_B200_LIB=$path timeout 120 python bench.py --no-cpu-baseline --workload $wl ${dt:+--dt $dt} --steps 20 --warmup 3 --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('$lib', d['config']['workload'], d['config']['dt'], '%.4g'%d['value'], '%.4g'%d['ms_per_step'])"
    done
  done
done
