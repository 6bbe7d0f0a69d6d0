mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "kernel_modes or every_window" > gpurun_out/g_parity.log 2>&1; echo parity rc=$?; tail -1 gpurun_out/g_parity.log
for w in ising2d_1024 ising1d_65536 noninteracting1d_1024x1000 ising1d_65536x64; do
  for G in 1 2 4; do
    for BS in 64 128 256; do
      [ $G = 1 ] && [ $BS != 64 ] && continue
      export KMC_GROUP=$G KMC_GROUP_BS=$BS
      timeout 120 python bench.py --no-cpu-baseline --workload $w --steps 50 --warmup 5 --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('$w G=$G bs=$BS', '%.4g'%d['value'], 'ms/step %.4g'%d['ms_per_step'], 'share %.3f'%d['roofline']['kernel_share_of_step'])"
    done
  done
done
