mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/final_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/final_tests.log
for w in ising2d_1024 ising1d_65536 noninteracting1d_1024x1000; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.log 2> gpurun_out/bench_$w.err; tail -1 gpurun_out/bench_$w.log > gpurun_out/bench_$w.json
  python -c "import json;d=json.load(open('gpurun_out/bench_$w.json'));print('$w', d['value'], d['e2e']['value'])"
done
