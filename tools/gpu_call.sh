mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "kernel_modes or full_size or sampled or maximum" > gpurun_out/tp.log 2>&1; echo tp rc=$?; tail -3 gpurun_out/tp.log
for r in 1 2; do for T in 0 1; do
for w in "ising2d_32768 --dt 0.01" "ising2d_32768 --dt 0.05" "ising2d_32768 --dt 0.003"; do
  KMC_TWOPASS=$T timeout 300 python bench.py --no-cpu-baseline --workload $w --steps 20 --warmup 3 --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('twopass=$T', d['config']['workload'], d['config']['dt'], '%.4g'%d['value'], 'su/s %.4g'%d['site_updates_per_s'])"
done; done; done
