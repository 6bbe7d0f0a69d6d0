mkdir -p gpurun_out
for r in 1 2; do for G in 2 4 8; do for BS in 64 128; do
  KMC_GROUP=$G KMC_GROUP_BS=$BS timeout 120 python bench.py --no-cpu-baseline --workload ising2d_1024 --steps 50 --warmup 5 --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('G=$G bs=$BS', d['config']['workload'], '%.4g'%d['value'])"
done; done; done
