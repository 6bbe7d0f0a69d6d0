mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_series.py -x -q > gpurun_out/pytest_hop.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_hop.log
for r in 1 2; do for hf in 1 0; do
  KMC_HOPFAST=$hf timeout 120 python bench.py --no-cpu-baseline --workload diff2d_8192 --steps 20 --warmup 3 --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('hopfast=$hf', d['config']['workload'], '%.4g'%d['value'], '%.4g'%d['ms_per_step'], d['roofline']['avg_launch_ms'])"
done; done
KMC_HOPLB=2 timeout 120 python bench.py --no-cpu-baseline --workload diff2d_8192 --steps 20 --warmup 3 --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('hoplb2', '%.4g'%d['value'], '%.4g'%d['ms_per_step'])"
