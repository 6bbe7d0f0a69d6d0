# parity of the ZGB grouped step + A/B against the generic ZGB step (KMC_ZGBFAST=0)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_zgb.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_zgb.log
for r in 1 2; do for zf in 1 0; do
  KMC_ZGBFAST=$zf timeout 120 python bench.py --no-cpu-baseline --workload zgb2d_32768 --steps 20 --warmup 3 --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('zgbfast=$zf', '%.4g'%d['value'], '%.4g'%d['ms_per_step'], '%.4g'%d['roofline']['avg_launch_ms'])"
done; done
