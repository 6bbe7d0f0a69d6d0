mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multigpu.py -m gpu -q -x -k "observables or vgroup or fused or loopback or uneven or maximum" > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gputests.log
for w in "ising2d_32768 --dt 0.01" "zgb2d_32768"; do
  timeout 300 python bench.py --no-cpu-baseline --workload $w --steps 30 --warmup 5 --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print(d['config']['workload'], d['config']['dt'], '%.4g'%d['value'], 'su/s %.4g'%d['site_updates_per_s'], 'ms %.4g'%d['ms_per_step'], 'share %.3f'%d['roofline']['kernel_share_of_step'])"
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --workload ising2d_32768 --dt 0.01"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches_obs.csv $CMD > /dev/null 2>&1; echo ncu rc=$?
for round in 1 2; do for L in abtmp/libkmc_qx8.so paper_1105_4673_b200/libkmc_b200.so; do
for w in "ising2d_32768" "ising2d_32768_strang" "ising2d_32768 --dt 0.01"; do
  KMC_B200_LIB=$L timeout 300 python bench.py --no-cpu-baseline --workload $w --steps 20 --warmup 3 --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('$L', d['config']['workload'], d['config']['dt'], '%.4g'%d['value'], 'ms %.4g'%d['ms_per_step'])"
done; done; done
