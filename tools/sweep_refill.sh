mkdir -p gpurun_out
KMC_REFILL=4 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_refill.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_refill.log
for r in 1 2 3 4 6 8; do
  for w in "ising2d_32768" "ising2d_32768 --dt 0.01" "zgb2d_32768" "diff2d_8192"; do
    KMC_REFILL=$r timeout 120 python bench.py --no-cpu-baseline --workload $w --steps 10 --warmup 3 --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('refill $r', d['config']['workload'], d['config']['dt'], '%.4g'%d['value'], '%.4g'%d['ms_per_step'])"
  done
done
