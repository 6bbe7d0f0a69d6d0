# refill-threshold sweep (KMC_REFILL) for the low-event workloads; prints events/s per setting
mkdir -p gpurun_out
for r in ${REFILLS:-4 8 12 16 24 32}; do
  for w in ${WORKLOADS:-"zgb2d_32768" "ising2d_32768:0.01"}; do
    wl=${w%%:*}; dt=${w#*:}; [ "$dt" = "$w" ] && dt=""
    KMC_REFILL=$r timeout 120 python bench.py --no-cpu-baseline --workload $wl ${dt:+--dt $dt} --steps 10 --warmup 3 --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('refill $r', d['config']['workload'], d['config']['dt'], '%.4g'%d['value'], '%.4g'%d['ms_per_step'])"
  done
done
