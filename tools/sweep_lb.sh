# register-cap / launch-shape variants (KMC_LB) x workloads, with the default refill rule
for lb in ${LBS:-0 5}; do
  for w in ${WORKLOADS:-"ising2d_32768" "ising2d_32768:0.01"}; do
    wl=${w%%:*}; dt=${w#*:}; [ "$dt" = "$w" ] && dt=""
    KMC_LB=$lb timeout 120 python bench.py --no-cpu-baseline --workload $wl ${dt:+--dt $dt} --steps 20 --warmup 3 --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('lb $lb', d['config']['workload'], d['config']['dt'], '%.4g'%d['value'], '%.4g'%d['ms_per_step'])"
  done
done
