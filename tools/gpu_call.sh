mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "every_window" > gpurun_out/lg.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/lg.log
for r in 1 2; do for L in abtmp/libkmc_base.so paper_1105_4673_b200/libkmc_b200.so; do
for w in ising2d_32768_strang ising2d_32768 "ising2d_32768 --dt 0.01"; do
  KMC_B200_LIB=$L timeout 300 python bench.py --no-cpu-baseline --workload $w --steps 20 --warmup 3 --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('$L', d['config']['workload'], d['config']['dt'], '%.4g'%d['value'])"
done; done; done
