# lanes-per-cell sweep (substep_group_kernel) on the small-lattice workloads; parity of every kernel mode first
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/g_parity.log 2>&1; echo parity rc=$?; tail -1 gpurun_out/g_parity.log
for w in ising2d_1024 ising1d_65536 ising1d_65536x64 noninteracting1d_1024x1000 ising2d_32768_strang; do
  for G in 1 2 4 8 16 32 auto; do
    if [ $G = auto ]; then unset KMC_GROUP; else export KMC_GROUP=$G; fi
    timeout 120 python bench.py --no-cpu-baseline --workload $w --steps 50 --warmup 5 --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('$w G=$G', '%.4g'%d['value'], 'ms/step %.4g'%d['ms_per_step'], d['clocks']['sm_mhz'])"
    [ $w = ising2d_32768_strang ] && break
  done
done
unset KMC_GROUP
