# quick GPU check used while tuning: parity tests, then the 4 main workloads (short runs)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_quick.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_quick.log
for w in "ising2d_32768" "ising2d_32768 --dt 0.01" "zgb2d_32768" "diff2d_8192"; do
  timeout 120 python bench.py --no-cpu-baseline --workload $w --steps 20 --warmup 3 --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print(d['config']['workload'], d['config']['dt'], '%.4g'%d['value'], '%.4g'%d['ms_per_step'], d['clocks']['sm_mhz'])"
done
