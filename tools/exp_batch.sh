# experiment batch: A/B of two builds on the spin-flip workloads + launch-shape variants of the
# diffusion block-walk kernel (KMC_HOPLB); short runs, outputs on stdout
WORKLOADS="ising2d_32768 ising2d_32768:0.01" bash tools/ab.sh
for r in 1 2; do for lb in 2 3 4; do
  KMC_B200_LIB=paper_1105_4673_b200/libkmc_b200_A.so KMC_HOPLB=$lb timeout 120 python bench.py --no-cpu-baseline --workload diff2d_8192 --steps 20 --warmup 3 --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('hoplb=$lb', '%.4g'%d['value'], '%.4g'%d['ms_per_step'])"
done; done
